# last verification of the committed tree: GPU suite, smoke, default bench, reference arm, launch list
set -x
O=gpurun_out/final5
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/bench_plain_for_ncu.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launches.log 2>&1
ls $O
