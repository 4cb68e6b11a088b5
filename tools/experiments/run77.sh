# in-sequence retune of configs 8/9; default bench (e2e path check)
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t77.tsv
timeout 2400 python -m paper_2208_09822_b200.tune --config 8 --config 9 --out gpurun_out/b200_t77.tsv --log gpurun_out/tune77.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t77.tsv paper_2208_09822_b200/tuning/b200.tsv
for c in 8 9; do timeout 900 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/bench77_c$c.json 2>gpurun_out/bench77_c$c.err; echo b$c=$?; done
timeout 900 python bench.py > gpurun_out/bench77.json 2>gpurun_out/bench77.err; echo bench=$?
