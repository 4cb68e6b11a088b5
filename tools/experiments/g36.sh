# producer order: first S chunks, C(u-1) store + C_in(u), rest (0) vs all chunks of u first (1)
set -x
for v in 0 1; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -DIAAT_KSG_PORDER=$v -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe_po$v tools/experiments/ksg_probe.cu
done
for i in 1 2; do for v in 0 1; do
timeout 300 gpurun_out/ksg_probe_po$v > gpurun_out/g36_po${v}_$i.log 2>&1
done; done
for v in 0 1; do echo "PORDER=$v"; grep -h "" gpurun_out/g36_po${v}_*.log | grep -v "_d[123]" | sort | sed -E 's/ +/ /g' | cut -d' ' -f1,10,11,16-18; done
