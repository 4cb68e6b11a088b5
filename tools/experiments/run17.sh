cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t17.tsv
timeout 2400 python -m paper_2208_09822_b200.tune --config 2 --min-n 48 --out gpurun_out/b200_t17.tsv --log gpurun_out/tune17.log > /dev/null 2>&1; echo tune=$?
