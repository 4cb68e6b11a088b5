K="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=4x8 IAAT_FORCE_ORDER=0 IAAT_FORCE_P=1 IAAT_FORCE_CTAS=3"
for d in 0 1 2 3; do env $K IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 64 64 64 --reps 8; done
K="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=4x8 IAAT_FORCE_ORDER=0 IAAT_FORCE_P=2 IAAT_FORCE_CTAS=2"
for d in 0 1 2 3; do env $K IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 64 64 64 --reps 8; done
K="IAAT_FORCE_FAMILY=2 IAAT_FORCE_TILE=5x8 IAAT_FORCE_ORDER=0 IAAT_FORCE_P=3 IAAT_FORCE_CTAS=1"
for d in 0 1 2 3; do env $K IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 80 80 80 --reps 8; done
for d in 0 1 2 3; do env $K IAAT_DEBUG_KS=$d python tools/run_case.py f32 NN 80 80 80 --reps 8 --beta 0; done
