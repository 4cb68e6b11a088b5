timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke50.log 2>&1; echo smoke=$?; cat gpurun_out/smoke50.log
i=0
for c in "f32 TT 68 68 68" "f32 NN 80 80 80" "f32 TT 76 76 76" "f32 NT 48 48 48"; do
  i=$((i+1))
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof50_$i python tools/run_case.py $c > gpurun_out/ncu50_$i.log 2>&1; echo ncu$i=$?
done
