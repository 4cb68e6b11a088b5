# ksg probe after hoisting the ragged chunk out of the chunk loop; KU variants
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe tools/experiments/ksg_probe.cu
timeout 300 gpurun_out/ksg_probe NN80 > gpurun_out/g30_probe.log 2>&1
timeout 300 gpurun_out/ksg_probe NN80 >> gpurun_out/g30_probe.log 2>&1
cat gpurun_out/g30_probe.log
