# multi-warp LDGSTS producers for misaligned (odd ld) K-streamed plans: parity + probe on config-3 shapes
timeout 900 python -m pytest tests -q -m gpu -x -k "ldgsts or ks_family" > gpurun_out/pytest65.log 2>&1; echo pytest=$?
timeout 1500 python tools/ldgsts_probe.py 37 67 79 67 67 17 61 67 31 37 47 79 79 31 53 31 61 61 > gpurun_out/run65.log 2>&1; echo probe=$?
