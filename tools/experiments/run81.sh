# FFMA2 pairs also for TN 16-byte-vector slab kernels
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "config4 or brute_force or integer or transpose or tn_extended" > gpurun_out/pytest81.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config 4 --no-e2e --no-cpu > gpurun_out/bench81_c4.json 2>gpurun_out/bench81_c4.err; echo b4=$?
timeout 900 python bench.py --config 8 --no-e2e --no-cpu > gpurun_out/bench81_c8.json 2>gpurun_out/bench81_c8.err; echo b8=$?
