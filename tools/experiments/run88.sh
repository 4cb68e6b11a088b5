# closing check of the committed tree
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest88.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke88.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench88.json 2>gpurun_out/bench88.err; echo bench=$?
