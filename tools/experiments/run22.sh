i=0
for spec in "IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=8x4 IAAT_FORCE_ORDER=5 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=3:f32 NN 64 64 64" \
            "IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=4x8 IAAT_FORCE_ORDER=0 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=3:f32 TT 64 64 64" \
            "IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=8x5 IAAT_FORCE_ORDER=3 IAAT_FORCE_P=3 IAAT_FORCE_CTAS=1:f32 NN 80 80 80"; do
  i=$((i+1))
  envs=${spec%%:*}; c=${spec#*:}
  env $envs python tools/run_case.py $c --plan > gpurun_out/case22_$i.log 2>&1
  env $envs timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof22_$i python tools/run_case.py $c > gpurun_out/ncu22_$i.log 2>&1; echo ncu$i=$?
done
