timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest53.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest53.log
for c in "f32 NN 37 67 79 100000" "f32 NN 31 61 61 100000" "f32 TN 29 29 29 500000" "f32 NN 67 67 17 100000"; do
  echo "default: $(python tools/run_case.py $c --alpha 1 --beta 1 2>&1 | tail -1)"
  for t in 4x8 4x4 8x4; do for P in 1 2; do for ct in 1 2 3; do
    r=$(IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=$t IAAT_FORCE_P=$P IAAT_FORCE_CTAS=$ct python tools/run_case.py $c --alpha 1 --beta 1 --plan 2>&1 | python3 -c 'import sys; L=sys.stdin.read().splitlines(); print(("ks" if "ks_fma" in L[0] or "ks1" in L[0] else "NOKS"), L[-1])')
    echo "  $t P$P c$ct: $r"
  done; done; done
done
