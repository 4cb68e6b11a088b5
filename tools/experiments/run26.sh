K="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=4x8 IAAT_FORCE_ORDER=0 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=3"
for d in 0 1 2 3; do env $K IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 64 64 64 --reps 8; done
K2="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=5x8 IAAT_FORCE_ORDER=0 IAAT_FORCE_P=3 IAAT_FORCE_CTAS=1"
for d in 0 2; do env $K2 IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 80 80 80 --reps 8; done
env $K IAAT_DEBUG_KS=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof26_1 python tools/run_case.py f32 NN 64 64 64 > /dev/null 2>&1; echo ncu1=$?
env $K timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof26_2 python tools/run_case.py f32 NN 64 64 64 > /dev/null 2>&1; echo ncu2=$?
