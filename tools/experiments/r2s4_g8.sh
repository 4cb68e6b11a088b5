# config-4 TN shapes below 0.70 (n = 19 slab, 23 / 26 / 27 ksgs): ncu --set full
O=gpurun_out/s4g8
mkdir -p $O
for n in 19 23 26 27 31; do
  python tools/run_case.py f32 TN $n $n $n 500000 --alpha -1 --beta 0.25 --reps 4 2>&1 | tail -1
done
for n in 19 26; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 2 -c 1 -o $O/prof_TN$n python tools/run_case.py f32 TN $n $n $n 500000 --alpha -1 --beta 0.25 > $O/ncu_TN$n.log 2>&1
done
ls $O
