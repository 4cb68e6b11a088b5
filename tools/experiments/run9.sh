for o in 0 1; do IAAT_FORCE_ORDER=$o timeout 120 python tools/sweep.py f32 NN 64 --tiles 4x4,4x8,8x8,8x4 --P 1,2 >> gpurun_out/sweep9.log 2>&1; done
for o in 0 1; do IAAT_FORCE_ORDER=$o timeout 120 python tools/sweep.py f32 TT 64 --tiles 4x4,4x8,8x8,8x4 --P 1,2 >> gpurun_out/sweep9.log 2>&1; done
for n in 16 32 48 80; do timeout 300 python tools/sweep.py f32 NN $n --tiles 8x8,4x8,8x4,4x4,8x2,2x8 --stage-kb 32,48,64,96 >> gpurun_out/sweep9.log 2>&1; done
for n in 32 48 80; do timeout 300 python tools/sweep.py f32 TT $n --tiles 8x8,4x8,8x4,4x4,8x2,2x8 --stage-kb 32,48,64,96 >> gpurun_out/sweep9.log 2>&1; done
