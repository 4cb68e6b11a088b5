nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -Ipaper_2208_09822_b200/csrc -o ksg_probe_bin tools/experiments/ksg_probe.cu || exit 1
timeout 300 ./ksg_probe_bin 2>&1 | tee gpurun_out/ksg3.log
