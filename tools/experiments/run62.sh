# full GPU suite + benches of configs 5, 7, 8, 9 with the merged tuning table
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest62.log 2>&1; echo pytest=$?
for c in 8 9 7 5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e > gpurun_out/bench62_c$c.json 2>gpurun_out/bench62_c$c.err; echo b$c=$?
done
