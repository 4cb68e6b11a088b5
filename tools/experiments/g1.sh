set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/peaks tools/peaks.cu && /tmp/peaks | tee gpurun_out/peaks.json
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -Ipaper_2208_09822_b200/csrc -o /tmp/ksg_probe tools/experiments/ksg_probe.cu && timeout 300 /tmp/ksg_probe 2>&1 | tee gpurun_out/ksg1.log
