timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest47.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest47.log
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t47.tsv
timeout 2400 python -m paper_2208_09822_b200.tune --config 2 --min-n 24 --out gpurun_out/b200_t47.tsv --log gpurun_out/tune47.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t47.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench47.json 2>gpurun_out/bench47.err; echo bench=$?
