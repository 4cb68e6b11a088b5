# round-1 closing evidence on the final tree: GPU tests, smoke, default bench, reference arm, launch list,
# ncu --set full of the dominant config-2 launch (TT 76)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest83.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke83.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench83.json 2>gpurun_out/bench83.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench83_ref.json 2>gpurun_out/bench83_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:iaat --csv --log-file gpurun_out/launches83.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu83_launch.log 2>&1; echo launches=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:iaat -s 3 -c 1 -o gpurun_out/prof83_TT76 python tools/run_case.py f32 TT 76 76 76 > /dev/null 2>&1; echo ncu=$?
