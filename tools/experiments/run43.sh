timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest43.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest43.log
for c in 6 7; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bench43_c$c.json 2>gpurun_out/bench43_c$c.err; echo bench$c=$?; done
