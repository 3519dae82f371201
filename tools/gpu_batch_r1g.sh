mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1g_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1g_smoke.log
timeout 900 python bench.py > gpurun_out/r1g_bench.json 2> gpurun_out/r1g_bench.err; echo "bench rc=$?" >> gpurun_out/r1g_bench.err
echo DONE
