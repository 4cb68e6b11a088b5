KS_PROBE_FAM=6 timeout 900 python tools/ks_probe.py f32 NN 64 f32 NT 64 f32 TT 64 f32 NN 48 f32 TT 48 f32 NN 72 f32 TT 72 f32 NN 80 > gpurun_out/ks46.log 2>&1; echo probe=$?
