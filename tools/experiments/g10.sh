# fp64 DMMA bank-conflict fix: fp64 parity, config-5 bench, ncu of the n=80 / n=64 NN launches
python -m pytest tests/test_gpu_parity.py -q -x -k "fp64 or config5 or ks_dmma or dmma or integer or transpose" 2>&1 | tail -3 | tee gpurun_out/g10_tests.log
python -m pytest tests/test_gpu_complex.py -q -x 2>&1 | tail -2 | tee -a gpurun_out/g10_tests.log
python bench.py --config 5 --steps 3 --warmup 1 --no-cpu > gpurun_out/g10_cfg5.json 2> gpurun_out/g10_cfg5.err
tail -c 700 gpurun_out/g10_cfg5.json
python tools/run_case.py f64 NN 80 80 80 200000 --beta 0 > gpurun_out/g10_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ksd -s 2 -c 1 -o gpurun_out/prof10_ksd_NN80 python tools/run_case.py f64 NN 80 80 80 200000 --beta 0 > gpurun_out/g10_ncu.log 2>&1
python tools/run_case.py f64 NN 64 64 64 200000 --beta 0 > gpurun_out/g10_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ksd -s 2 -c 1 -o gpurun_out/prof10_ksd_NN64 python tools/run_case.py f64 NN 64 64 64 200000 --beta 0 > gpurun_out/g10_ncu2.log 2>&1
