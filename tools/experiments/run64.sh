# C staged through smem (TMA load/store) in the K-streamed FMA kernels: parity + timing vs run59/63
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest64.log 2>&1; echo pytest=$?
for sh in "NT 64" "TT 64" "NT 80" "TT 80" "NT 56" "TT 72" "NN 64"; do set -- $sh
  timeout 60 python tools/run_case.py f32 $1 $2 $2 $2 --reps 6 --plan | tr '\n' ' ' | grep -o '"family": "[a-z0-9_]*"\|"c_staged": [0-9]\|f32 .*GFLOP/s'; echo
done > gpurun_out/run64.log 2>&1
