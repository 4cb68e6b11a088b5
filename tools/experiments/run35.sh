timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest35.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest35.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench35.json 2>gpurun_out/bench35.err; echo bench=$?
