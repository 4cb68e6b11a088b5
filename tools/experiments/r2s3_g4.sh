# ncu of the tuned ksgs plans of config-3's top shapes
set -x
mkdir -p gpurun_out/g4
python tools/run_case.py f32 NN 37 67 79 100000 --reps 2 --alpha 1 --beta 1 --plan > gpurun_out/g4/plan.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iaat_ksgs -s 1 -c 1 -o gpurun_out/g4/ksgs_37x67x79 python tools/run_case.py f32 NN 37 67 79 100000 --reps 2 --alpha 1 --beta 1 > gpurun_out/g4/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iaat_ksgs -s 1 -c 1 -o gpurun_out/g4/ksgs_61x67x31 python tools/run_case.py f32 NN 61 67 31 100000 --reps 2 --alpha 1 --beta 1 > gpurun_out/g4/ncu2.log 2>&1
tail -3 gpurun_out/g4/ncu1.log gpurun_out/g4/ncu2.log
