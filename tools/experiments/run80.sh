# FFMA2 pairs for TN scalar-load (odd ld) slab kernels: parity + config 4 / 8 benches
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "config4 or brute_force or integer or transpose or misaligned or tn_extended" > gpurun_out/pytest80.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config 4 --no-e2e --no-cpu > gpurun_out/bench80_c4.json 2>gpurun_out/bench80_c4.err; echo b4=$?
timeout 900 python bench.py --config 8 --no-e2e --no-cpu > gpurun_out/bench80_c8.json 2>gpurun_out/bench80_c8.err; echo b8=$?
