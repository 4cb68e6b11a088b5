timeout 900 python -m pytest tests/test_gpu_complex.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest56.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest56.log
for n in 16 32 48 64 80; do
  echo "c64 NN $n default: $(python tools/run_case.py c64 NN $n $n $n --reps 6 2>&1 | tail -1)"
done
