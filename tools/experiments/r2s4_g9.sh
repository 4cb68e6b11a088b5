# ksgs: per-row address registers (no IMAD per row per k-step): parity, configs 3 / 4
set -x
O=gpurun_out/s4g9
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_ksg.py -m gpu -x -q > $O/pytest_ksg.log 2>&1; echo "rc $?" >> $O/pytest_ksg.log
tail -4 $O/pytest_ksg.log
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 600 python bench.py --config 10 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg10.json 2> $O/bench_cfg10.err
for c in 3 4 10; do python -c "
import json
d=json.loads(open('$O/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])
low=[(s['shape'],s['frac_roofline']) for s in d['shapes'] if s['frac_roofline']<0.70]
print(len(low), low)"; done
