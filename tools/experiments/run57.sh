timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest57.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest57.log
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t57.tsv
timeout 1800 python -m paper_2208_09822_b200.tune --config 7 --out gpurun_out/b200_t57.tsv --log gpurun_out/tune57.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t57.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --config 7 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench57_c7.json 2>gpurun_out/bench57_c7.err; echo bench7=$?
