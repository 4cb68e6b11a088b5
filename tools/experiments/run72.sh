# retune config 2 (n >= 36) with in-sequence timing (a separator call before each timed call), then bench
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t72.tsv
timeout 3000 python -m paper_2208_09822_b200.tune --config 2 --min-n 36 --out gpurun_out/b200_t72.tsv --log gpurun_out/tune72.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t72.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench72.json 2>gpurun_out/bench72.err; echo bench=$?
