timeout 800 python tools/ks_probe.py f32 NN 80 f32 TT 80 f32 NN 64 f32 TT 64 f32 NT 64 f32 NN 48 f32 TT 48 f32 NN 36 f32 TT 36 > gpurun_out/ks23.log 2>&1; echo probe=$?
