# wider tile grid retune for config 3's large shapes (min(M, N) >= 48 gets the extra tiles); bench
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t91.tsv
timeout 2000 python -m paper_2208_09822_b200.tune --config 3 --min-n 48 --out gpurun_out/b200_t91.tsv --log gpurun_out/tune91.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t91.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --config 3 --no-e2e --no-cpu > gpurun_out/bench91_c3.json 2>gpurun_out/bench91_c3.err; echo b3=$?
