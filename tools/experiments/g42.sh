# ksgr (slab staging + in-smem repack): parity, then forced vs current plan on odd / misaligned shapes
set -x
timeout 900 python -m pytest tests/test_gpu_ksg.py -x -q -k "ksgr or ksgs" > gpurun_out/g42_pytest.log 2>&1; echo "rc $?" >> gpurun_out/g42_pytest.log
tail -3 gpurun_out/g42_pytest.log
run() { python tools/run_case.py "$@" 2>&1 | tail -1; IAAT_FORCE_FAMILY=9 python tools/run_case.py "$@" 2>&1 | tail -1; }
for s in "37 67 79" "67 67 17" "53 31 47" "47 53 17" "79 31 53" "31 61 61" "61 67 31"; do
  run f32 NN $s 100000 --alpha 1 --beta 1
done > gpurun_out/g42_cfg3.log
for n in 19 23 26 27 30 31; do
  run f32 TN $n $n $n 500000 --alpha -1 --beta 0.25
done > gpurun_out/g42_cfg4.log
for n in 38 42 62 66 78; do for tr in NN TT; do run f32 $tr $n $n $n --alpha 1.5 --beta 0.5; done; done > gpurun_out/g42_heldout.log
cat gpurun_out/g42_cfg3.log gpurun_out/g42_cfg4.log gpurun_out/g42_heldout.log
