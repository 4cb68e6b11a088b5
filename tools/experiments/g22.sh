for ef in 1 0; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -DIAAT_KSG_EVICT_FIRST=$ef -Ipaper_2208_09822_b200/csrc -o ksg_probe_bin$ef tools/experiments/ksg_probe.cu || exit 1
echo "== evict_first=$ef"; timeout 300 ./ksg_probe_bin$ef 2>&1
done
