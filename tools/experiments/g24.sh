for sh in "TT 76 3872" "NN 76 3872" "NT 68 4837"; do
  set -- $sh
  python tools/run_case.py f32 $1 $2 $2 $2 $3 --plan > gpurun_out/g24_plain_$1$2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ksg -s 2 -c 1 -o gpurun_out/prof24_$1$2 python tools/run_case.py f32 $1 $2 $2 $2 $3 > gpurun_out/g24_ncu_$1$2.log 2>&1
done
