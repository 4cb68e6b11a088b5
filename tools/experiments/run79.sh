# L1 prefetch of C_in during the last K-chunk (K-streamed fp32, MN-major rows): config-2 bench
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ks_family or config2" > gpurun_out/pytest79.log 2>&1; echo pytest=$?
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench79.json 2>gpurun_out/bench79.err; echo bench=$?
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench79b.json 2>gpurun_out/bench79b.err; echo bench=$?
