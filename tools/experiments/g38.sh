# round 2 session 2: GPU suite after the KU=1 fix; ksg retune with the KU=1 entries; config 2 + 5 bench
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g38_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g38_pytest.log
tail -2 gpurun_out/g38_pytest.log
timeout 1500 python -m paper_2208_09822_b200.tune --config 2 --ksg --min-n 36 --log gpurun_out/g38_tune_ksg.log > gpurun_out/g38_tune_ksg.out 2>&1
timeout 900 python -m paper_2208_09822_b200.tune --config 2 --min-n 28 --max-n 28 --log gpurun_out/g38_tune28.log > gpurun_out/g38_tune28.out 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g38.tsv
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g38_cfg2.json 2> gpurun_out/g38_cfg2.err
timeout 600 python bench.py --config 5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/g38_cfg5.json 2> gpurun_out/g38_cfg5.err
tail -c 300 gpurun_out/g38_cfg2.json
