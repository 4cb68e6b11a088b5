for sh in "NN 56 7133" "NT 56 7133" "TT 56 7133"; do
  set -- $sh
  python tools/run_case.py f32 $1 $2 $2 $2 $3 --plan > gpurun_out/g21_plain_$1$2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ksg -s 2 -c 1 -o gpurun_out/prof21_$1$2 python tools/run_case.py f32 $1 $2 $2 $2 $3 > gpurun_out/g21_ncu_$1$2.log 2>&1
done
