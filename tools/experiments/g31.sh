# FFMA2 microbenchmark with the ksg NN fragment shape; KU=1 fix check
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/ffma2_order tools/experiments/ffma2_order.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe tools/experiments/ksg_probe.cu
timeout 120 gpurun_out/ffma2_order > gpurun_out/g31_micro.log 2>&1
timeout 300 gpurun_out/ksg_probe k16u1 > gpurun_out/g31_probe.log 2>&1
cat gpurun_out/g31_micro.log gpurun_out/g31_probe.log
