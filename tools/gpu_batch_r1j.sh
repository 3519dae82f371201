mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1j_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1j_smoke.log
timeout 900 python bench.py > gpurun_out/r1j_bench.json 2> gpurun_out/r1j_bench.err; echo "bench rc=$?" >> gpurun_out/r1j_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1j_bench_ref.json 2> gpurun_out/r1j_bench_ref.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r1j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1j_pytest.log
echo DONE
