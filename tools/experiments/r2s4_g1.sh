# round 2 session 4: HEAD verification (GPU suite, smoke, bench configs 2/3/4)
set -x
O=gpurun_out/s4g1
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc $?" >> $O/smoke.log
timeout 900 python bench.py --no-cpu --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
for f in $O/bench_cfg*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])
low=[(s['shape'],s['frac_roofline']) for s in d['shapes'] if s['frac_roofline']<0.70]
print(len(low), low)"; done
