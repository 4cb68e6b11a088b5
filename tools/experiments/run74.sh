# programmatic dependent launch: parity, config 1/2/3/4 with and without (IAAT_NO_PDL=1)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest74.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke74.log 2>&1; echo smoke=$?
for c in 2 1 3 4; do
  timeout 900 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/bench74_c$c.json 2>gpurun_out/bench74_c$c.err; echo b$c=$?
  IAAT_NO_PDL=1 timeout 900 python bench.py --config $c --no-e2e --no-cpu > gpurun_out/bench74_c${c}_nopdl.json 2>gpurun_out/bench74_c${c}_nopdl.err; echo b${c}n=$?
done
