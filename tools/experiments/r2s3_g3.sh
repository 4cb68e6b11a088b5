# ksgs with C through the stage (span store by the producer): parity, sweep, retune config 3/4, benches
set -x
L=paper_2208_09822_b200
mkdir -p gpurun_out/g3
timeout 900 python -m pytest tests/test_gpu_ksg.py -q -x -k ksgs > gpurun_out/g3/pytest.log 2>&1; r=$?; tail -15 gpurun_out/g3/pytest.log; [ $r = 0 ] || exit 1
cp gpurun_out/g1/b200_after.tsv $L/tuning/b200.tsv
timeout 900 python tools/experiments/ksgs_sweep.py NN 37x67x79 37x47x79 61x67x31 67x61x7 > gpurun_out/g3/sweep.log 2>&1
timeout 1500 python -m $L.tune --config 3 --config 4 --ksg --log gpurun_out/g3/tune_ksg.log > /dev/null 2>&1
cp $L/tuning/b200.tsv gpurun_out/g3/b200_after.tsv
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g3/cfg3.json 2> gpurun_out/g3/cfg3.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g3/cfg4.json 2> gpurun_out/g3/cfg4.err
