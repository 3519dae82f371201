# round-2 batch ae: L2 prefetch of the fused epilogues' operands (A/B), scratch pool retention (e2e phases), GPU suite
bash tools/ab_bench.sh tools/ab_pf0.so tools/ab_pf1.so 3 > gpurun_out/r2ae_ab64.txt 2>&1
bash tools/ab_bench_fp32.sh tools/ab_pf0.so tools/ab_pf1.so 2 > gpurun_out/r2ae_ab32.txt 2>&1
HPR_VERBOSE=1 python tools/time_e2e.py fp32 > gpurun_out/r2ae_e2e32.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r2ae_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2ae_pytest.log
