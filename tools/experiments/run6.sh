for n in 8 16 32; do timeout 300 python tools/sweep.py f32 NN $n --tiles 8x8,4x8,4x4,2x8,8x2,2x4,4x2,2x2 --stage-kb 24,40,52,72,100 --S 2,3,4 >> gpurun_out/sweep6.log 2>&1; done
for n in 48 64; do timeout 300 python tools/sweep.py f32 NN $n --tiles 8x8,4x8,8x4,4x4,2x8,8x6,6x8,4x6 --P 1,2,3 --S 2,3,4 >> gpurun_out/sweep6.log 2>&1; done
timeout 300 python tools/sweep.py f32 NN 80 --tiles 8x8,4x8,8x4,4x4,5x8,8x5,4x5,5x4 --P 1,2 --S 2,3 >> gpurun_out/sweep6.log 2>&1
timeout 300 python tools/sweep.py f32 TT 64 --tiles 8x8,4x8,8x4,4x4 --P 1,2 --S 2,3,4 >> gpurun_out/sweep6.log 2>&1
timeout 300 python tools/sweep.py f32 NT 64 --tiles 8x8,4x8,8x4,4x4 --P 1,2 --S 2,3,4 >> gpurun_out/sweep6.log 2>&1
