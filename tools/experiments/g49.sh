# bench with per-shape times from back-to-back runs of each call
set -x
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g49_cfg2.json 2> gpurun_out/g49_cfg2.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g49_cfg4.json 2> gpurun_out/g49_cfg4.err
for f in gpurun_out/g49_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['config'].get('per_call_sum_ms'), d['config'].get('per_call_sequence_sum_ms'), d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])
low=[(s['shape'],s['frac_roofline']) for s in d['shapes'] if s['frac_roofline']<0.70 and int(s['shape'].split('_')[2].split('x')[0])>=16]
print(len(low), low)"; done
