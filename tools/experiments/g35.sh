# C out through global stores from registers (IAAT_KSG_C_STG=1) vs C through smem + TMA store (0)
set -x
for v in 0 1; do
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -DIAAT_KSG_C_STG=$v -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe_cs$v tools/experiments/ksg_probe.cu
done
for i in 1 2; do for v in 0 1; do
timeout 300 gpurun_out/ksg_probe_cs$v > gpurun_out/g35_cs${v}_$i.log 2>&1
done; done
for v in 0 1; do echo "C_STG=$v"; grep -h "" gpurun_out/g35_cs${v}_*.log | grep -v "_d[123]" | sort | sed -E 's/ +/ /g' | cut -d' ' -f1,10,11,16-18; done
