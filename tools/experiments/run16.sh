timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest16.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest16.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench16.json 2>gpurun_out/bench16.err; echo bench=$?
for s in 2 4; do for pad in 0 100000; do IAAT_DEBUG_SMEM_PAD=$pad IAAT_FORCE_CTAS=1 timeout 120 python tools/sweep.py f32 NN 64 --tiles 4x8 --P 1 --S $s >> gpurun_out/sweep16.log 2>&1; done; done
cat gpurun_out/sweep16.log
