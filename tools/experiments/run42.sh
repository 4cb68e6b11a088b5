timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches42.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch42.log 2>&1; echo ncu_launch=$?
i=0
for c in "f32 TT 68 68 68" "f32 TT 76 76 76" "f32 NN 80 80 80" "f32 NT 64 64 64" "f32 NN 16 16 16" "f64 NN 64 64 64 32768 --beta 0 --alpha 1"; do
  i=$((i+1))
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof42_$i python tools/run_case.py $c > gpurun_out/ncu42_$i.log 2>&1; echo ncu$i=$?
done
