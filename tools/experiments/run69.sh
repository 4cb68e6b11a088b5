# wider slab knob grid on the slowest config-2 shapes
timeout 2400 python tools/slab_probe.py TT 68 TT 76 NN 76 NN 80 NT 76 TT 72 NN 68 NT 68 > gpurun_out/run69.log 2>&1; echo probe=$?
