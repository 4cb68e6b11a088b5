# ncu of three ksg probe variants (one launch each, after a plain run of the same command)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -Ipaper_2208_09822_b200/csrc -o ksg_probe_bin tools/experiments/ksg_probe.cu || exit 1
for v in NN64_8x8_l4_g2w4_p2 TT64_8x8_l4_g2w4_p2 NN80_10x5_l4_g2w4_p1; do
  ./ksg_probe_bin $v > gpurun_out/plain_$v.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:kprobe -s 2 -c 1 -o gpurun_out/prof_$v ./ksg_probe_bin $v > gpurun_out/ncu_$v.log 2>&1
done
ls -la gpurun_out
