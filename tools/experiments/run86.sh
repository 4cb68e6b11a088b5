# ZGEMM epilogue: C_in loads of block pairs before their stores
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "complex" > gpurun_out/pytest86.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config 7 --no-e2e --no-cpu > gpurun_out/bench86_c7.json 2>gpurun_out/bench86_c7.err; echo b7=$?
