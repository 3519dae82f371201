# round-2 batch ad: where the FP32 e2e time goes (fused vs split), per-phase host times
for f in 1 0; do
  HPR_FUSED=$f HPR_VERBOSE=1 python tools/time_e2e.py fp32 > gpurun_out/r2ad_e2e32_f$f.log 2>&1
done
HPR_VERBOSE=1 python tools/time_e2e.py fp64 > gpurun_out/r2ad_e2e64_f1.log 2>&1
