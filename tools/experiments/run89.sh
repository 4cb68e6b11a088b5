# wider first-strip tile grid (3, 5, 6) in the tuner for fp32 n >= 48; retune config 2 (n >= 48) and bench
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t89.tsv
timeout 2400 python -m paper_2208_09822_b200.tune --config 2 --min-n 48 --out gpurun_out/b200_t89.tsv --log gpurun_out/tune89.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t89.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench89.json 2>gpurun_out/bench89.err; echo bench=$?
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench89b.json 2>gpurun_out/bench89b.err; echo bench=$?
