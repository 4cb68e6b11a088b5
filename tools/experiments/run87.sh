# retune config 7 (ZGEMM) with the paired C_in epilogue; bench
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t87.tsv
timeout 1800 python -m paper_2208_09822_b200.tune --config 7 --out gpurun_out/b200_t87.tsv --log gpurun_out/tune87.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t87.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --config 7 --no-e2e --no-cpu > gpurun_out/bench87_c7.json 2>gpurun_out/bench87_c7.err; echo b7=$?
