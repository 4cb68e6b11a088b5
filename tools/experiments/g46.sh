# A/B again with the clean-timing bench (events only at the ends of the timed region, PDL overlap intact):
# L2 prefetch of the first units before griddepcontrol.wait (pf) vs without (base)
set -x
L=paper_2208_09822_b200
cp $L/libiaat.so /tmp/libiaat_pf.so
gunzip -c $L/libiaat_base.so.gz > /tmp/libiaat_base.so
for r in 1 2; do
for v in base pf; do
  cp /tmp/libiaat_$v.so $L/libiaat.so
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g46_cfg2_${v}_$r.json 2> gpurun_out/g46_cfg2_${v}_$r.err
  timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g46_cfg4_${v}_$r.json 2> gpurun_out/g46_cfg4_${v}_$r.err
done
done
cp /tmp/libiaat_pf.so $L/libiaat.so
for f in gpurun_out/g46_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
