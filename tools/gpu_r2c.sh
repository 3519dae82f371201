./tools/flow_probe.bin > gpurun_out/r2c_flow.log 2>&1
