# retune configs 3 and 4 over the ksg / ksgs catalog (new g3w4 small-tile entries), then bench them
O=gpurun_out/s4g11
mkdir -p $O
timeout 2400 python -m paper_2208_09822_b200.tune --ksg --config 4 --config 3 --log $O/tune_ksgs.log > /dev/null 2>&1
echo "tune rc $?"
cp paper_2208_09822_b200/tuning/b200.tsv $O/b200.tsv
grep -c "^ksg" $O/tune_ksgs.log
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
for c in 3 4; do python -c "
import json
d=json.loads(open('$O/bench_cfg$c.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])
low=[(s['shape'],s['frac_roofline']) for s in d['shapes'] if s['frac_roofline']<0.70]
print(len(low), low)"; done
