timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest10.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest10.log
for c in 1 2; do for n in 32 48 64 80; do IAAT_FORCE_CTAS=$c timeout 300 python tools/sweep.py f32 NN $n --tiles 8x8,4x8,8x4,4x4,4x6,6x4 --stage-kb 24,32,48,64,96 >> gpurun_out/sweep10.log 2>&1; done; done
for c in 1 2; do for n in 48 64 80; do IAAT_FORCE_CTAS=$c timeout 300 python tools/sweep.py f32 TT $n --tiles 8x8,4x8,8x4,4x4 --stage-kb 24,32,48,64,96 >> gpurun_out/sweep10.log 2>&1; done; done
