# retune config 2 (n >= 36) with explicit C_in staging trials + re-timed leaders, then bench
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t70.tsv
timeout 3000 python -m paper_2208_09822_b200.tune --config 2 --min-n 36 --out gpurun_out/b200_t70.tsv --log gpurun_out/tune70.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t70.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench70.json 2>gpurun_out/bench70.err; echo bench=$?
