# pair-register A fragments (no float->pair repacking): probe
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -DIAAT_KSG_PAIR_FRAGS=0 -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe_pf0 tools/experiments/ksg_probe.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -DIAAT_KSG_PAIR_FRAGS=1 -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe_pf1 tools/experiments/ksg_probe.cu
for i in 1 2; do
timeout 300 gpurun_out/ksg_probe_pf0 NN > gpurun_out/g33_pf0_$i.log 2>&1
timeout 300 gpurun_out/ksg_probe_pf1 NN > gpurun_out/g33_pf1_$i.log 2>&1
done
grep -h "OK" gpurun_out/g33_pf0_*.log | sort; echo ---; grep -h "OK" gpurun_out/g33_pf1_*.log | sort
