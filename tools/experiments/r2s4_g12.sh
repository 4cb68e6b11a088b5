# 8x8 ksg tiles on three consumer warpgroups: parity, config-2 retune of n = 44..64 over the ksg catalog, bench
O=gpurun_out/s4g12
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_ksg.py -m gpu -x -q -k "ksg_every_entry or column_pair" > $O/pytest_ksg.log 2>&1; echo "rc $?" >> $O/pytest_ksg.log
tail -3 $O/pytest_ksg.log
cp paper_2208_09822_b200/tuning/b200.tsv $O/b200_before.tsv
timeout 1800 python -m paper_2208_09822_b200.tune --ksg --config 2 --min-n 44 --max-n 64 --log $O/tune_ksg.log > /dev/null 2>&1
echo "tune rc $?"
cp paper_2208_09822_b200/tuning/b200.tsv $O/b200.tsv
grep "^ksg" $O/tune_ksg.log | cut -c1-170
timeout 900 python bench.py --no-cpu --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python -c "
import json
d=json.loads(open('$O/bench_cfg2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])
low=[(s['shape'],s['frac_roofline']) for s in d['shapes'] if s['frac_roofline']<0.70]
print(len(low), low)"
