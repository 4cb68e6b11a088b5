# pipelined ragged-chunk pieces: ksg parity, then config-2 bench and the n = 76 / 78 / 80 timings
set -x
O=gpurun_out/s4g7
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_ksg.py -m gpu -x -q > $O/pytest_ksg.log 2>&1; echo "rc $?" >> $O/pytest_ksg.log
tail -4 $O/pytest_ksg.log
timeout 900 python bench.py --no-cpu --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python -c "
import json
d=json.loads(open('$O/bench_cfg2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['clocks'])
low=[(s['shape'],s['frac_roofline']) for s in d['shapes'] if s['frac_roofline']<0.70]
print(len(low), low)"
for n in 76 78 80; do for tr in NN NT TT; do
  e=0; [ $tr = NT ] && e=6; [ $tr = TT ] && e=12
  IAAT_FORCE_FAMILY=7 IAAT_FORCE_ORDER=$e python tools/run_case.py f32 $tr $n $n $n --reps 6 2>&1 | tail -1
done; done
