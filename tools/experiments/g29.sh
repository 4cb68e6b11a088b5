# ncu of the ksg compute-only loop (d3) vs the FFMA2 microbenchmark; fp64 n=8/16 tuning
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gpurun_out/ffma2_order tools/experiments/ffma2_order.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe tools/experiments/ksg_probe.cu
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kprobe -s 1 -c 1 -o gpurun_out/prof29_d3 gpurun_out/ksg_probe NN80_10x10_l4_k16u2_g4w2_p1_s2_d3 > gpurun_out/g29_ncu_d3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kprobe -s 1 -c 1 -o gpurun_out/prof29_d0 gpurun_out/ksg_probe NN80_10x10_l4_k16u2_g4w2_p1_s2 > gpurun_out/g29_ncu_d0.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kord -s 31 -c 1 -o gpurun_out/prof29_micro gpurun_out/ffma2_order > gpurun_out/g29_ncu_micro.log 2>&1
timeout 1200 python -m paper_2208_09822_b200.tune --config 5 --max-n 16 --log gpurun_out/g29_tune5.log > gpurun_out/g29_tune5.out 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g29.tsv
