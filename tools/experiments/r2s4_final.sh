# round 2 session 4 closing evidence: GPU suite, smoke, default bench (+ e2e, cpu baseline), reference arm,
# configs 3/4/5, launch list of the bench command, ncu --set full of the dominant config-2 launches
set -x
O=gpurun_out/final4
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg5.json 2> $O/bench_cfg5.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/bench_plain_for_ncu.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launches.log 2>&1
for sh in "NT 76 3872" "TT 76 3872" "NN 76 3872" "NT 68 4837"; do
  set -- $sh
  python tools/run_case.py f32 $1 $2 $2 $2 $3 > $O/plain_$1$2.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 2 -c 1 -o $O/prof_$1$2 python tools/run_case.py f32 $1 $2 $2 $2 $3 > $O/ncu_$1$2.log 2>&1
done
ls $O
