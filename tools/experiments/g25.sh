python -m pytest tests/test_gpu_parity.py -q -x -k "ks_dmma or config5 or fp64" 2>&1 | tail -2
for tr in NN NT; do
for n in 80 64; do
  echo "== $tr $n table"; python tools/run_case.py f64 $tr $n $n $n 700000 --beta 0 --reps 6
  for t in 40x40 32x40 40x32 32x32; do
    echo "== $tr $n forced $t"; IAAT_FORCE_FAMILY=3 IAAT_FORCE_TILE=$t python tools/run_case.py f64 $tr $n $n $n 700000 --beta 0 --reps 6
  done
done
done
