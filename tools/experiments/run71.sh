timeout 600 python tools/context_probe.py > gpurun_out/run71.log 2>&1; echo probe=$?
