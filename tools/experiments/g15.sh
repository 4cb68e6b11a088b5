python -m pytest tests/test_gpu_ksg.py tests/test_gpu_parity.py -q -x -k "ksg or config2_full" 2>&1 | tail -2 | tee gpurun_out/g15_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/g15_bench.json 2> gpurun_out/g15_bench.err
tail -c 200 gpurun_out/g15_bench.json
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/g15_plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/g15_ncu_launch.log 2>&1
for sh in "NN 76 3872" "TT 76 3872" "NN 68 4837" "TT 80 3495"; do
  set -- $sh
  python tools/run_case.py f32 $1 $2 $2 $2 $3 > gpurun_out/g15_plain_$1$2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ksg -s 2 -c 1 -o gpurun_out/prof15_$1$2 python tools/run_case.py f32 $1 $2 $2 $2 $3 > gpurun_out/g15_ncu_$1$2.log 2>&1
done
