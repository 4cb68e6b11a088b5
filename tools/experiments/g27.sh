python -m paper_2208_09822_b200.tune --config 5 --max-n 16 --log gpurun_out/g27_tune5.log > gpurun_out/g27_tune5.out 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g27.tsv
tail -5 gpurun_out/g27_tune5.log
