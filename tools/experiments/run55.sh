timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest55.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest55.log
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t55.tsv
timeout 1800 python -m paper_2208_09822_b200.tune --config 6 --out gpurun_out/b200_t55.tsv --log gpurun_out/tune55.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t55.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --config 6 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench55_c6.json 2>gpurun_out/bench55_c6.err; echo bench6=$?
