timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest41.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest41.log
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t41.tsv
timeout 2400 python -m paper_2208_09822_b200.tune --config 2 --config 1 --config 4 --config 3 --out gpurun_out/b200_t41.tsv --log gpurun_out/tune41.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t41.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench41.json 2>gpurun_out/bench41.err; echo bench=$?
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench41_c$c.json 2>gpurun_out/bench41_c$c.err; echo bench$c=$?; done
