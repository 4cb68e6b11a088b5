K="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=4x8 IAAT_FORCE_ORDER=0 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=3"
env $K IAAT_DEBUG_KS=6 timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof30_1 python tools/run_case.py f32 NN 64 64 64 > /dev/null 2>&1; echo ncu1=$?
