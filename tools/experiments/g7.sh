# ksg: parity tests, ksg-vs-current retune of config 2 (n >= 36), config-2 bench
python -m pytest tests/test_gpu_ksg.py -x -q 2>&1 | tail -3 | tee gpurun_out/g7_ksg_tests.log
python -m paper_2208_09822_b200.tune --config 2 --ksg --min-n 36 --log gpurun_out/g7_tune.log > /dev/null 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g7.tsv
python -m pytest tests/test_gpu_parity.py -x -q -k "config2_full" 2>&1 | tail -2 | tee gpurun_out/g7_c2full.log
python bench.py --steps 10 --warmup 3 > gpurun_out/g7_bench.json 2> gpurun_out/g7_bench.err
tail -c 300 gpurun_out/g7_bench.json
