# in-sequence retune of config 2 (n < 36), configs 3 and 4; benches
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t73.tsv
timeout 1500 python -m paper_2208_09822_b200.tune --config 2 --max-n 35 --out gpurun_out/b200_t73.tsv --log gpurun_out/tune73.log > /dev/null 2>&1; echo tune2=$?
timeout 1800 python -m paper_2208_09822_b200.tune --config 4 --out gpurun_out/b200_t73.tsv --log gpurun_out/tune73.log > /dev/null 2>&1; echo tune4=$?
timeout 2400 python -m paper_2208_09822_b200.tune --config 3 --out gpurun_out/b200_t73.tsv --log gpurun_out/tune73.log > /dev/null 2>&1; echo tune3=$?
cp gpurun_out/b200_t73.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench73_c2.json 2>gpurun_out/bench73_c2.err; echo b2=$?
timeout 900 python bench.py --config 3 --no-e2e --no-cpu > gpurun_out/bench73_c3.json 2>gpurun_out/bench73_c3.err; echo b3=$?
timeout 900 python bench.py --config 4 --no-e2e --no-cpu > gpurun_out/bench73_c4.json 2>gpurun_out/bench73_c4.err; echo b4=$?
