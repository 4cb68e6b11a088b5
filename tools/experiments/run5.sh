timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest5.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest5.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench5.json 2>gpurun_out/bench5.err; echo bench=$?
for n in 8 16 32 48 64 80; do timeout 200 python tools/sweep.py f32 NN $n --P 1,2,3,4,6,8,12,16 >> gpurun_out/sweep5.log 2>&1; done
timeout 200 python tools/sweep.py f32 NN 64 --tiles 8x8,4x8,8x4,4x4 --P 1,2,3,4 >> gpurun_out/sweep5.log 2>&1
timeout 200 python tools/sweep.py f32 NN 80 --tiles 8x8,8x5,5x8,4x8 --P 1,2 >> gpurun_out/sweep5.log 2>&1
