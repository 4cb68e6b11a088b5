timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest44.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest44.log
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench44_c1.json 2>gpurun_out/bench44_c1.err; echo bench1=$?
timeout 600 python bench.py --config 3 --grouped --steps 5 --warmup 3 > gpurun_out/bench44_c3g.json 2>gpurun_out/bench44_c3g.err; echo bench3g=$?
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t44.tsv
timeout 1800 python -m paper_2208_09822_b200.tune --config 6 --config 7 --out gpurun_out/b200_t44.tsv --log gpurun_out/tune44.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t44.tsv paper_2208_09822_b200/tuning/b200.tsv
for c in 6 7; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bench44_c$c.json 2>gpurun_out/bench44_c$c.err; echo bench$c=$?; done
