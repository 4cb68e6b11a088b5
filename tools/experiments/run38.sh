timeout 600 python tools/ks_probe.py f32 NN 80 f32 TT 80 f32 NN 64 f32 TT 64 f32 NT 64 > gpurun_out/ks38.log 2>&1; echo probe=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench38.json 2>gpurun_out/bench38.err; echo bench=$?
