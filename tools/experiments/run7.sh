timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest7.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest7.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench7.json 2>gpurun_out/bench7.err; echo bench=$?
timeout 300 python tools/sweep.py f32 TT 64 --tiles 8x8,4x8,8x4,4x4 --P 1,2 >> gpurun_out/sweep7.log 2>&1
IAAT_FORCE_ORDER=0 timeout 300 python tools/sweep.py f32 TT 64 --tiles 8x8,4x8 --P 2 >> gpurun_out/sweep7.log 2>&1
IAAT_FORCE_ORDER=1 timeout 300 python tools/sweep.py f32 TT 64 --tiles 8x8,4x8 --P 2 >> gpurun_out/sweep7.log 2>&1
for c in 1 2; do IAAT_FORCE_CTAS=$c timeout 300 python tools/sweep.py f32 NN 32 --tiles 8x8,4x8,4x4 --P 2,3,4,5,6,8 >> gpurun_out/sweep7.log 2>&1; done
for c in 1 2; do IAAT_FORCE_CTAS=$c timeout 300 python tools/sweep.py f32 NN 64 --tiles 8x8,4x8,4x4 --P 1,2 >> gpurun_out/sweep7.log 2>&1; done
