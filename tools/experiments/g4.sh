nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -Ipaper_2208_09822_b200/csrc -o ksg_probe_bin tools/experiments/ksg_probe.cu || exit 1
for v in NN80_10x5_l4_g2w4_p1 TT64_8x8_l8_g2w2_p1 NT64_8x8_l4_g2w4_p2; do
  ./ksg_probe_bin $v > gpurun_out/plain_$v.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:kprobe -s 2 -c 1 -o gpurun_out/prof4_$v ./ksg_probe_bin $v > gpurun_out/ncu4_$v.log 2>&1
done
