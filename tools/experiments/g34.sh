nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/ffma2_morph tools/experiments/ffma2_morph.cu
timeout 120 gpurun_out/ffma2_morph
