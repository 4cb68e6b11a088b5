# tighter LDGSTS producer loops (hoisted params, 4-row unroll): parity + probe
timeout 900 python -m pytest tests -q -m gpu -x -k "ldgsts or ks_family" > gpurun_out/pytest67.log 2>&1; echo pytest=$?
timeout 1500 python tools/ldgsts_probe.py 37 67 79 67 67 17 61 67 31 37 47 79 > gpurun_out/run67.log 2>&1; echo probe=$?
