# ksgs entries x ring depths on the worst config-3 shapes; ncu of 37x67x79 on its tuned plan
set -x
mkdir -p gpurun_out/g2
timeout 900 python tools/experiments/ksgs_sweep.py NN 37x67x79 37x47x79 79x31x53 61x67x31 31x37x37 > gpurun_out/g2/sweep.log 2>&1
cp gpurun_out/g1/b200_after.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iaat_ksgs -c 1 -o gpurun_out/g2/ksgs_37x67x79 python tools/run_case.py f32 NN 37 67 79 100000 --reps 2 --alpha 1 --beta 1 > gpurun_out/g2/ncu.log 2>&1
tail -3 gpurun_out/g2/ncu.log
