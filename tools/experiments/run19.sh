timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest19.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest19.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench19.json 2>gpurun_out/bench19.err; echo bench=$?
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench19_c$c.json 2>gpurun_out/bench19_c$c.err; echo bench$c=$?; done
