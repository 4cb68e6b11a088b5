python -m pytest tests -q -m gpu -x 2>&1 | tail -4 | tee gpurun_out/g18_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -9 | tee gpurun_out/g18_smoke.log
python bench.py > gpurun_out/g18_bench.json 2> gpurun_out/g18_bench.err
tail -c 250 gpurun_out/g18_bench.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g18_ref.json 2> gpurun_out/g18_ref.err
tail -c 300 gpurun_out/g18_ref.json
