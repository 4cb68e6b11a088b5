timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest92.log 2>&1; echo pytest=$?
