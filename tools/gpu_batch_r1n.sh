mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_screen.py -m gpu -q > gpurun_out/r1n_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1n_pytest.log
timeout 120 python -c "
from paper_2510_10891_b200 import screen
print([round(screen.fp64_peak_tflops(),2) for _ in range(3)])" > gpurun_out/r1n_peak.log 2>&1
timeout 900 python bench.py > gpurun_out/r1n_bench.json 2> gpurun_out/r1n_bench.err; echo "bench rc=$?" >> gpurun_out/r1n_bench.err
echo DONE
