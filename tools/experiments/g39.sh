# ncu of the config-4 TN shapes below 0.70 (current tuned plans)
set -x
for n in 19 23 26 27; do
  python tools/run_case.py f32 TN $n $n $n 500000 --alpha -1 --beta 0.25 > gpurun_out/g39_plain_$n.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 2 -c 1 -o gpurun_out/prof39_TN$n python tools/run_case.py f32 TN $n $n $n 500000 --alpha -1 --beta 0.25 > gpurun_out/g39_ncu_$n.log 2>&1
done
