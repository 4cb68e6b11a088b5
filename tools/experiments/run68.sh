# round-1 final evidence with the current tree: GPU tests, smoke, default bench (+ reference arm),
# launch list of the bench command, ncu --set full of the largest config-2 launches
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest68.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke68.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench68.json 2>gpurun_out/bench68.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench68_ref.json 2>gpurun_out/bench68_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:iaat --csv --log-file gpurun_out/launches68.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu68_launch.log 2>&1; echo launches=$?
for sh in "TT 68" "TT 76" "NN 76"; do set -- $sh
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof68_$1$2 python tools/run_case.py f32 $1 $2 $2 $2 > /dev/null 2>&1; echo ncu$1$2=$?
done
