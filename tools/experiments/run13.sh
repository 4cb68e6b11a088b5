for c in 1 2; do for s in 2 3 4; do IAAT_FORCE_CTAS=$c IAAT_FORCE_S=$s timeout 120 python tools/sweep.py f32 NN 64 --tiles 4x8 --P 1 >> gpurun_out/sweep13.log 2>&1; done; done
for c in 1 2; do for s in 2 3 4; do IAAT_FORCE_CTAS=$c IAAT_FORCE_S=$s timeout 120 python tools/sweep.py f32 NN 32 --tiles 4x8 --P 2,4 >> gpurun_out/sweep13.log 2>&1; done; done
for c in 1 2; do for s in 2 3 4; do IAAT_FORCE_CTAS=$c IAAT_FORCE_S=$s timeout 120 python tools/sweep.py f32 NN 16 --tiles 4x4 --P 5,10 >> gpurun_out/sweep13.log 2>&1; done; done
