python bench.py --config 5 --steps 3 --warmup 1 --no-cpu > gpurun_out/g26_cfg5.json 2> gpurun_out/g26_cfg5.err
python -c "
import json
d=json.loads(open('gpurun_out/g26_cfg5.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['kernel'], d['roofline']['frac'])
for s in d['shapes']: print(s['shape'], s['ms'], s['gflops'], s['frac_roofline'])
"
python tools/run_case.py f64 NN 80 80 80 200000 --beta 0 > gpurun_out/g26_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ksd -s 2 -c 1 -o gpurun_out/prof26_ksd_NN80 python tools/run_case.py f64 NN 80 80 80 200000 --beta 0 > gpurun_out/g26_ncu.log 2>&1
