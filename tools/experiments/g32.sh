# FFMA2 microbenchmark: data-dependent power?  (i%7 data vs uniform random floats), with clocks sampled
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/ffma2_order tools/experiments/ffma2_order.cu
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv -lms 100 > gpurun_out/g32_smi.csv 2>&1 &
SMI=$!
sleep 1
timeout 120 gpurun_out/ffma2_order > gpurun_out/g32_micro.log 2>&1
sleep 1; kill $SMI; true
cat gpurun_out/g32_micro.log; sort gpurun_out/g32_smi.csv | uniq -c | sort -rn | head -20
