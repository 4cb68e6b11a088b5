python -m pytest tests/test_gpu_parity.py -q -x -k "elongated or grouped" 2>&1 | tail -3 | tee gpurun_out/g9_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -8 | tee gpurun_out/g9_smoke.log
python bench.py --config 5 --steps 3 --warmup 1 --no-cpu > gpurun_out/g9_cfg5.json 2> gpurun_out/g9_cfg5.err
tail -c 400 gpurun_out/g9_cfg5.json
python tools/heldout.py --out gpurun_out/heldout_r02.json > gpurun_out/g9_heldout.log 2>&1
tail -2 gpurun_out/g9_heldout.log
