python -m pytest tests/test_gpu_parity.py -q -x -k "shards_bitwise" 2>&1 | tail -2 | tee gpurun_out/g19_tests.log
nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/host_overhead.cu -Iinclude -Lpaper_2208_09822_b200 -liaat -Xlinker -rpath=$PWD/paper_2208_09822_b200 -o /tmp/host_overhead && /tmp/host_overhead | tee gpurun_out/host_overhead_r02.json
