# bench with events only at the ends of the timed region (PDL overlap kept) vs the per-call breakdown pass
set -x
for r in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g45_cfg2_$r.json 2> gpurun_out/g45_cfg2_$r.err
done
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g45_cfg4.json 2> gpurun_out/g45_cfg4.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g45_cfg3.json 2> gpurun_out/g45_cfg3.err
for f in gpurun_out/g45_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], 'sum per-call ms', round(sum(s['us'] for s in d['shapes'])/1e3,4), d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])"; done
