# retune config 4 with the FFMA2 TN scalar kernels; bench
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t82.tsv
timeout 1800 python -m paper_2208_09822_b200.tune --config 4 --out gpurun_out/b200_t82.tsv --log gpurun_out/tune82.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t82.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --config 4 --no-e2e --no-cpu > gpurun_out/bench82_c4.json 2>gpurun_out/bench82_c4.err; echo b4=$?
