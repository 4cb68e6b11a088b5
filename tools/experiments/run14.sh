timeout 2400 python -m paper_2208_09822_b200.tune --config 2 --out gpurun_out/b200_cfg2.tsv --log gpurun_out/tune_cfg2.log > /dev/null 2>&1; echo tune=$?
tail -3 gpurun_out/tune_cfg2.log
