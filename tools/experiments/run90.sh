timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest90.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke90.log 2>&1; echo smoke=$?
