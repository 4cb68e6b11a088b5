for cfg in "4x8 0 1 3" "4x8 0 3 1" "8x4 5 1 3" "4x4 0 1 4" "4x4 0 2 2"; do
set -- $cfg
K="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=$1 IAAT_FORCE_ORDER=$2 IAAT_FORCE_P=$3 IAAT_FORCE_CTAS=$4"
for d in 0 2 6; do echo "$cfg dbg $d: $(env $K IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 64 64 64 --reps 8 --plan 2>&1 | python3 -c 'import sys; L=sys.stdin.read().splitlines(); print(L[0][:40] if L else "", L[-1])')"; done
done
