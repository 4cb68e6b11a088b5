# round-1 session-3 evidence pass: gpu tests, bench (N=1), launch list, ncu full of two kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi20.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest20.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest20.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke20.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench20.json 2>gpurun_out/bench20.err; echo bench=$?
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench20_c$c.json 2>gpurun_out/bench20_c$c.err; echo bench$c=$?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches20.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch20.log 2>&1; echo ncu_launch=$?
i=0
for c in "f32 NN 16 16 16" "f32 NN 80 80 80" "f32 TT 64 64 64" "f64 NN 64 64 64"; do
  i=$((i+1))
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof20_$i python tools/run_case.py $c > gpurun_out/ncu20_$i.log 2>&1; echo ncu$i=$?
done
