# FFMA2 source order of the pair-fragment kernels (1 pair-outer, 2 snake, 3 scalar-outer, 4 scalar-outer snake)
set -x
for o in 1 2 3 4; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -DIAAT_KSG_PF_ORDER=$o -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe_o$o tools/experiments/ksg_probe.cu &
done; wait
for i in 1 2; do for o in 1 2 3 4; do
timeout 300 gpurun_out/ksg_probe_o$o N > gpurun_out/g37_o${o}_$i.log 2>&1
done; done
for o in 1 2 3 4; do echo "ORDER=$o"; grep -h "" gpurun_out/g37_o${o}_*.log | grep -v "_d[123]" | sort | sed -E 's/ +/ /g' | cut -d' ' -f1,10,11,16-18; done
