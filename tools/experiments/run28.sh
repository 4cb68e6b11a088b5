for t in 4x8 4x4 8x4; do
K="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=$t IAAT_FORCE_ORDER=0 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=3"
for d in 0 2 6 3; do echo "tile $t dbg $d: $(env $K IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 64 64 64 --reps 8)"; done
done
