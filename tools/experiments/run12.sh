timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "config2_square or config3_irregular or brute" > gpurun_out/pytest12.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest12.log
for o in 0 3 5 9 17; do for n in 48 64 80; do IAAT_FORCE_ORDER=$o timeout 300 python tools/sweep.py f32 NN $n --tiles 8x8,4x8,8x4,6x8,8x6 --P 1,2,3 >> gpurun_out/sweep12_o$o.log 2>&1; done; done
for o in 1 3 5 9 17; do for n in 64; do IAAT_FORCE_ORDER=$o timeout 300 python tools/sweep.py f32 TT $n --tiles 8x8,4x8,8x4 --P 1,2 >> gpurun_out/sweep12_tt_o$o.log 2>&1; done; done
