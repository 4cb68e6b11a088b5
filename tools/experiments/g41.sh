# ksgs with C_in staged in the slab stage: parity tests, config 4 / 3 bench
set -x
timeout 900 python -m pytest tests/test_gpu_ksg.py -x -q -k ksgs > gpurun_out/g41_pytest.log 2>&1; echo "rc $?" >> gpurun_out/g41_pytest.log
tail -3 gpurun_out/g41_pytest.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g41_cfg4.json 2> gpurun_out/g41_cfg4.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g41_cfg3.json 2> gpurun_out/g41_cfg3.err
IAAT_FORCE_CSMEM=0 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g41_cfg4_nocs.json 2> gpurun_out/g41_cfg4_nocs.err
for f in gpurun_out/g41_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['roofline']['kernel'], d['roofline']['frac'])
print([(s['shape'].split('_')[2], s['frac_roofline']) for s in d['shapes'] if s['frac_roofline'] < 0.7])"; done
