# FLOP / DRAM audit of single launches (ncu counters)
timeout 2400 python tools/audit.py run gpurun_out/audit76 > gpurun_out/audit76.log 2>&1; echo audit=$?
