# ksg family: parity tests, then ksg-vs-current tuning of config 2 (n >= 36), then the config-2 bench
python -m pytest tests/test_gpu_ksg.py -x -q 2>&1 | tail -5 | tee gpurun_out/g6_ksg_tests.log
python -m pytest tests/test_gpu_parity.py -x -q -k "config2_full" 2>&1 | tail -3 | tee gpurun_out/g6_c2full.log
python -m paper_2208_09822_b200.tune --config 2 --ksg --min-n 36 --log gpurun_out/g6_tune.log > /dev/null 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g6.tsv
python bench.py --steps 10 --warmup 3 > gpurun_out/g6_bench.json 2> gpurun_out/g6_bench.err
tail -c 600 gpurun_out/g6_bench.json
