timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench48.json 2>gpurun_out/bench48.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench48_ref.json 2>gpurun_out/bench48_ref.err; echo ref=$?
