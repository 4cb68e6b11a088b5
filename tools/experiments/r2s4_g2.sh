# round 2 session 4: column-pair TMA boxes (ksg PV) -- parity tests, then the held-out sweep
set -x
O=gpurun_out/s4g2
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_ksg.py -m gpu -x -q -k "column_pair" > $O/pytest_pv.log 2>&1; echo "rc $?" >> $O/pytest_pv.log
tail -30 $O/pytest_pv.log
if grep -q "rc 0" $O/pytest_pv.log; then
  timeout 1500 python tools/heldout.py --out $O/heldout.json > $O/heldout.log 2>&1
  head -33 $O/heldout.log | cut -c1-200
  tail -3 $O/heldout.log | cut -c1-400
fi
