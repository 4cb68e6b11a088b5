# full GPU suite + smoke on the current tree
python -m pytest tests -q -m gpu -x 2>&1 | tail -15 | tee gpurun_out/g8_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -8 | tee gpurun_out/g8_smoke.log
