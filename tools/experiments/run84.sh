# one pass over environ for the knob key instead of seven getenv calls: full GPU suite + config 1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest84.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config 1 --no-e2e --no-cpu > gpurun_out/bench84_c1.json 2>gpurun_out/bench84_c1.err; echo b1=$?
timeout 900 python bench.py --config 1 --no-e2e --no-cpu > gpurun_out/bench84_c1b.json 2>gpurun_out/bench84_c1b.err; echo b1=$?
