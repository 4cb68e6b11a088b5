python -m pytest tests/test_gpu_ksg.py -q -x 2>&1 | tail -3 | tee gpurun_out/g12_tests.log
python -m paper_2208_09822_b200.tune --config 3 --ksg --log gpurun_out/g12_tune3.log > /dev/null 2>&1
cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_g12.tsv
python bench.py --config 3 --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/g12_cfg3.json 2> gpurun_out/g12_cfg3.err
tail -c 300 gpurun_out/g12_cfg3.json
python tools/heldout.py --out gpurun_out/heldout_r02b.json > gpurun_out/g12_heldout.log 2>&1
tail -1 gpurun_out/g12_heldout.log
