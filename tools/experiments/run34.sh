timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest34.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest34.log
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t34.tsv
timeout 1800 python -m paper_2208_09822_b200.tune --config 2 --min-n 20 --out gpurun_out/b200_t34.tsv --log gpurun_out/tune34.log > /dev/null 2>&1; echo tune=$?
