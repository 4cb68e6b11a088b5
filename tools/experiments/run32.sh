for t in 4x8 8x4 4x4 4x6; do
K="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=$t IAAT_FORCE_ORDER=0 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=3"
for d in 0 6; do echo "tile $t dbg $d: $(env $K IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 64 64 64 --reps 8 2>&1 | tail -1)"; done
done
