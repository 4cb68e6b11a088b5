# dependent-call chain test; in-sequence retune of the complex sweeps (configs 6, 7) and benches
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "dependent_calls or integer_inputs" > gpurun_out/pytest75.log 2>&1; echo pytest=$?
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t75.tsv
timeout 2400 python -m paper_2208_09822_b200.tune --config 6 --config 7 --out gpurun_out/b200_t75.tsv --log gpurun_out/tune75.log > /dev/null 2>&1; echo tune=$?
cp gpurun_out/b200_t75.tsv paper_2208_09822_b200/tuning/b200.tsv
for c in 6 7; do timeout 900 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/bench75_c$c.json 2>gpurun_out/bench75_c$c.err; echo b$c=$?; done
