# 7-block DMMA warp tiles (M or N = 56): parity, retune n=56 (configs 7, 9), bench 7/9
timeout 1200 python -m pytest tests -q -m gpu -k "tn_extended or ks_dmma or complex" > gpurun_out/pytest61.log 2>&1; echo pytest=$?
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t61.tsv
timeout 1200 python -m paper_2208_09822_b200.tune --config 7 --config 9 --min-n 56 --max-n 56 --out gpurun_out/b200_t61.tsv --log gpurun_out/tune61.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t61.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 600 python bench.py --config 9 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench61_c9.json 2>gpurun_out/bench61_c9.err; echo b9=$?
timeout 600 python bench.py --config 7 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench61_c7.json 2>gpurun_out/bench61_c7.err; echo b7=$?
