set -e
for c in "f32 NN 8 8 8" "f32 NN 32 32 32" "f32 TT 64 64 64" "f32 NN 80 80 80" "f32 NN 4 4 4"; do
  python tools/run_case.py $c --plan >> gpurun_out/plain_cases.log 2>&1
done
i=0
for c in "f32 NN 8 8 8" "f32 NN 32 32 32" "f32 TT 64 64 64" "f32 NN 80 80 80" "f32 NN 4 4 4"; do
  i=$((i+1))
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof_$i python tools/run_case.py $c > gpurun_out/ncu_$i.log 2>&1
done
