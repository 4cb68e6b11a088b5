# config 4 (TN) retune on the current library (full pass for n >= 16, then the ksg/ksgs pass), then bench
set -x
timeout 2400 python -m paper_2208_09822_b200.tune --config 4 --min-n 16 --log gpurun_out/g50_tune4.log > gpurun_out/g50_tune4.out 2>&1
timeout 1200 python -m paper_2208_09822_b200.tune --config 4 --ksg --log gpurun_out/g50_tune4_ksg.log > gpurun_out/g50_tune4_ksg.out 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g50.tsv
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g50_cfg4.json 2> gpurun_out/g50_cfg4.err
tail -40 gpurun_out/g50_tune4.log; tail -25 gpurun_out/g50_tune4_ksg.log
