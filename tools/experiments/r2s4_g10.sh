# ksgs entries with three consumer warpgroups (g3w4): parity, then forced against the current plans
O=gpurun_out/s4g10
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_ksg.py -m gpu -x -q -k ksgs > $O/pytest_ksgs.log 2>&1; echo "rc $?" >> $O/pytest_ksgs.log
tail -3 $O/pytest_ksgs.log
run() { python tools/run_case.py "$@" 2>&1 | tail -1; }
for n in 15 17 19 21 22 23 25 26 27 29 30 31; do
  echo "== TN $n"
  run f32 TN $n $n $n 500000 --alpha -1 --beta 0.25 --reps 5
  for e in 30 31 32; do
    echo -n "  e$e: "; IAAT_FORCE_FAMILY=8 IAAT_FORCE_ORDER=$e run f32 TN $n $n $n 500000 --alpha -1 --beta 0.25 --reps 5
  done
done > $O/tn_sweep.log 2>&1
cat $O/tn_sweep.log
for sh in "31 23 53" "23 37 11" "47 23 7" "31 37 37" "17 37 61" "13 37 61" "31 11 79" "11 53 11" "17 17 7"; do
  set -- $sh
  echo "== NN $1 $2 $3"
  run f32 NN $1 $2 $3 100000 --alpha 1 --beta 1 --reps 5
  for e in 33 34 35; do
    echo -n "  e$e: "; IAAT_FORCE_FAMILY=8 IAAT_FORCE_ORDER=$e run f32 NN $1 $2 $3 100000 --alpha 1 --beta 1 --reps 5
  done
done > $O/nn_sweep.log 2>&1
cat $O/nn_sweep.log
