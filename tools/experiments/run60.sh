# TN above 32^3 (extended domain) + fp64 TN/TT -- parity, tuning, bench
timeout 900 python -m pytest tests -q -m gpu -k "tn_extended or fp64_other or ks_dmma" > gpurun_out/pytest60.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config 8 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench60_c8_pre.json 2>gpurun_out/bench60_c8_pre.err; echo b8pre=$?
timeout 600 python bench.py --config 9 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench60_c9_pre.json 2>gpurun_out/bench60_c9_pre.err; echo b9pre=$?
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t60.tsv
timeout 2400 python -m paper_2208_09822_b200.tune --config 8 --config 9 --out gpurun_out/b200_t60.tsv --log gpurun_out/tune60.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t60.tsv paper_2208_09822_b200/tuning/b200.tsv
timeout 600 python bench.py --config 8 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench60_c8.json 2>gpurun_out/bench60_c8.err; echo b8=$?
timeout 600 python bench.py --config 9 --steps 5 --warmup 3 --no-e2e > gpurun_out/bench60_c9.json 2>gpurun_out/bench60_c9.err; echo b9=$?
