# beta=0.5 vs beta=0 on the large config-2 shapes: how much does the C_in read cost?
for tr in NN NT TT; do for n in 56 64 68 72 76 80; do
  for b in 0.5 0; do timeout 60 python tools/run_case.py f32 $tr $n $n $n --reps 6 --beta $b; done
done; done > gpurun_out/run59.log 2>&1
