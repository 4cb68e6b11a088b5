for o in 0 1; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -DIAAT_KSG_FMA_ORDER=$o -Ipaper_2208_09822_b200/csrc -o ksg_probe_bin$o tools/experiments/ksg_probe.cu || exit 1
echo "== FMA order $o"; timeout 300 ./ksg_probe_bin$o 2>&1
done
