timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest37.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest37.log
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t37.tsv
timeout 1800 python -m paper_2208_09822_b200.tune --config 5 --out gpurun_out/b200_t37.tsv --log gpurun_out/tune37.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t37.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench37_c5.json 2>gpurun_out/bench37_c5.err; echo bench5=$?
