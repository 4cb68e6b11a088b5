# ncu of the ksgr kernels (TN 19^3, NN 37x67x79)
set -x
export IAAT_FORCE_FAMILY=9
python tools/run_case.py f32 TN 19 19 19 500000 --alpha -1 --beta 0.25 > gpurun_out/g43_plain_tn19.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ksgr -s 2 -c 1 -o gpurun_out/prof43_tn19 python tools/run_case.py f32 TN 19 19 19 500000 --alpha -1 --beta 0.25 > gpurun_out/g43_ncu1.log 2>&1
python tools/run_case.py f32 NN 37 67 79 100000 --alpha 1 --beta 1 --plan > gpurun_out/g43_plain_nn37.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ksgr -s 2 -c 1 -o gpurun_out/prof43_nn37 python tools/run_case.py f32 NN 37 67 79 100000 --alpha 1 --beta 1 > gpurun_out/g43_ncu2.log 2>&1
