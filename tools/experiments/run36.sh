timeout 800 python tools/ks_probe.py f64 NN 64 f64 NT 64 f64 NN 80 f64 NT 80 f64 NN 48 f64 NN 32 > gpurun_out/ks36.log 2>&1; echo probe=$?
