# column-pair boxes vs the same entry on aligned shapes (timing), ncu --set full of NN 78 / TT 78 (PV)
O=gpurun_out/s4g6
mkdir -p $O
for n in 76 78 80; do for tr in NN NT TT; do
  e=0; [ $tr = NT ] && e=6; [ $tr = TT ] && e=12
  IAAT_FORCE_FAMILY=7 IAAT_FORCE_ORDER=$e python tools/run_case.py f32 $tr $n $n $n --reps 6 --plan 2>&1 | cut -c1-600 >> $O/time.log
done; done
cat $O/time.log | grep -v "^{" 
for tr in NN TT; do
  IAAT_FORCE_FAMILY=7 timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 2 -c 1 -o $O/prof_${tr}78 python tools/run_case.py f32 $tr 78 78 78 > $O/ncu_${tr}78.log 2>&1
done
e=0
IAAT_FORCE_FAMILY=7 IAAT_FORCE_ORDER=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 2 -c 1 -o $O/prof_NN80_e0 python tools/run_case.py f32 NN 80 80 80 > $O/ncu_NN80.log 2>&1
ls -la $O
