# round 2 session 3: ksgs on one shared ring (+ odd-shape entries, odd tiles on FFMA2):
# parity of every ksgs entry (incl. ring wrap), then config 3 / 4 ksgs retune and benches
set -x
L=paper_2208_09822_b200
mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_ksg.py -q -x -k ksgs > gpurun_out/g1/pytest.log 2>&1; r=$?; tail -15 gpurun_out/g1/pytest.log; [ $r = 0 ] || exit 1
cp $L/tuning/b200.tsv gpurun_out/g1/b200_before.tsv
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g1/cfg3_before.json 2> gpurun_out/g1/cfg3_before.err
timeout 1500 python -m $L.tune --config 3 --config 4 --ksg --log gpurun_out/g1/tune_ksg.log > /dev/null 2>&1
cp $L/tuning/b200.tsv gpurun_out/g1/b200_after.tsv
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g1/cfg3_after.json 2> gpurun_out/g1/cfg3_after.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g1/cfg4_after.json 2> gpurun_out/g1/cfg4_after.err
for f in gpurun_out/g1/cfg*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
