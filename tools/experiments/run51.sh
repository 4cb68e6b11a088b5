cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t51.tsv
timeout 2400 python -m paper_2208_09822_b200.tune --config 4 --config 3 --out gpurun_out/b200_t51.tsv --log gpurun_out/tune51.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t51.tsv paper_2208_09822_b200/tuning/b200.tsv
for c in 3 4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench51_c$c.json 2>gpurun_out/bench51_c$c.err; echo bench$c=$?; done
