python -m pytest tests/test_gpu_ksg.py -q -x -k ksgs 2>&1 | tail -3 | tee gpurun_out/g16_tests.log
python -m paper_2208_09822_b200.tune --config 4 --ksg --log gpurun_out/g16_tune4.log > gpurun_out/g16_tune4.out 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g16.tsv
python bench.py --config 4 --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/g16_cfg4.json 2> gpurun_out/g16_cfg4.err
tail -c 300 gpurun_out/g16_cfg4.json
