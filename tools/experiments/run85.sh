# ncu --set full of the fp64 config-5 dominant launch (NN 80, K-streamed DMMA) and the ZGEMM 80 launch
timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof85_f64NN80 python tools/run_case.py f64 NN 80 80 80 200000 --alpha 1 --beta 0 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof85_c64NT80 python tools/run_case.py c64 NT 80 80 80 > /dev/null 2>&1; echo ncu2=$?
