export IAAT_FORCE_TILE=4x8 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=2
python tools/run_case.py f32 NN 64 64 64 --plan > gpurun_out/case11.log 2>&1 && timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof11 python tools/run_case.py f32 NN 64 64 64 > gpurun_out/ncu11.log 2>&1
