# ksgs double-buffered fragments: parity + sweep; held-out sweep with and without ksgs as the misaligned default
set -x
L=paper_2208_09822_b200
mkdir -p gpurun_out/g5
timeout 900 python -m pytest tests/test_gpu_ksg.py -q -x -k ksgs > gpurun_out/g5/pytest.log 2>&1; r=$?; tail -5 gpurun_out/g5/pytest.log; [ $r = 0 ] || exit 1
timeout 900 python tools/experiments/ksgs_sweep.py NN 37x67x79 37x47x79 61x67x31 > gpurun_out/g5/sweep.log 2>&1
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g5/cfg3.json 2> gpurun_out/g5/cfg3.err
timeout 1200 python tools/heldout.py --out gpurun_out/g5/heldout_slab.json > gpurun_out/g5/heldout_slab.log 2>&1
IAAT_KSGS_DEFAULT=1 timeout 1200 python tools/heldout.py --out gpurun_out/g5/heldout_ksgs.json > gpurun_out/g5/heldout_ksgs.log 2>&1
