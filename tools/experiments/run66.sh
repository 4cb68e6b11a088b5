# ncu of the LDGSTS K-streamed kernel (forced) on a config-3 shape
export IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=6x4 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=2 IAAT_FORCE_NPW=2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof66 python tools/run_case.py f32 NN 37 67 79 100000 --alpha 1 --beta 1 > gpurun_out/ncu66.log 2>&1; echo ncu=$?
