python -m paper_2208_09822_b200.tune --config 3 --ksg --log gpurun_out/g13_tune3.log > gpurun_out/g13_tune3.out 2>&1
tail -20 gpurun_out/g13_tune3.out
python tools/run_case.py f32 NN 38 38 38 > gpurun_out/g13_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ksgs -s 2 -c 1 -o gpurun_out/prof13_ksgs_NN38 python tools/run_case.py f32 NN 38 38 38 > gpurun_out/g13_ncu.log 2>&1
