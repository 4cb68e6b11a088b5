O=gpurun_out/s4g4
mkdir -p $O
export CUDA_LAUNCH_BLOCKING=1
for tr in NN TT; do
  echo "== $tr" >> $O/log.txt
  timeout 120 python tools/run_case.py f32 $tr 38 38 38 2000 --reps 2 --beta 0.5 >> $O/log.txt 2>&1
  echo "rc $?" >> $O/log.txt
done
grep -v "^  \|^Traceback\|File" $O/log.txt | cut -c1-250
