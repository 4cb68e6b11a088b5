python -m pytest tests/test_gpu_ksg.py tests/test_gpu_parity.py -q -x -k "ksg or ks_ or dmma or config5" 2>&1 | tail -2 | tee gpurun_out/g23_tests.log
python -m paper_2208_09822_b200.tune --config 2 --ksg --min-n 36 --log gpurun_out/g23_tune.log > gpurun_out/g23_tune.out 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g23.tsv
python bench.py --steps 20 --warmup 5 > gpurun_out/g23_bench.json 2> gpurun_out/g23_bench.err
python bench.py --config 5 --steps 3 --warmup 1 --no-cpu > gpurun_out/g23_cfg5.json 2> gpurun_out/g23_cfg5.err
python -c "
import json
for f in ['gpurun_out/g23_bench.json','gpurun_out/g23_cfg5.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['roofline']['kernel'], d['roofline']['frac'])
"
