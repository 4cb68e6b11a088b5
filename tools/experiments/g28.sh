# round 2 session 2: FFMA2 order / bank model vs measured; ksg time split; GPU suite; config 5 + 2
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/ffma2_order tools/experiments/ffma2_order.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/ffma2_rf tools/experiments/ffma2_rf.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/ffma2_lds tools/experiments/ffma2_lds.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -lcuda -Ipaper_2208_09822_b200/csrc -o gpurun_out/ksg_probe tools/experiments/ksg_probe.cu
(timeout 120 gpurun_out/ffma2_order; timeout 60 gpurun_out/ffma2_rf; timeout 60 gpurun_out/ffma2_lds) > gpurun_out/g28_micro.log 2>&1
timeout 300 gpurun_out/ksg_probe NN80 > gpurun_out/g28_probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g28_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g28_pytest.log
timeout 600 python bench.py --config 5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/g28_cfg5.json 2> gpurun_out/g28_cfg5.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g28_cfg2.json 2> gpurun_out/g28_cfg2.err
tail -3 gpurun_out/g28_pytest.log
