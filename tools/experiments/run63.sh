# how much of a K-streamed unit is the epilogue? IAAT_DEBUG_KS=2 skips it (timing only)
for sh in "NT 64" "TT 64" "NT 80" "TT 80" "NT 56" "TT 72"; do set -- $sh
  for d in 0 2 1; do echo "dbg=$d"; IAAT_DEBUG_KS=$d timeout 60 python tools/run_case.py f32 $1 $2 $2 $2 --reps 6 --plan | tail -1; done
done > gpurun_out/run63.log 2>&1
