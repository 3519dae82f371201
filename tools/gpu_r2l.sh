# round-2 batch l: row-panel test, full C4 bench record, C5 bench with e2e, C4 FP32 bench
python -m pytest tests/test_gpu_variants.py -x -q > gpurun_out/r2l_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2l_pytest.log
python bench.py > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
python bench.py --config C5 --steps 10 --warmup 3 --no-screen --no-cpu-baseline > gpurun_out/r2l_c5.json 2> gpurun_out/r2l_c5.err
python bench.py --precision fp32 --no-screen > gpurun_out/r2l_fp32.json 2> gpurun_out/r2l_fp32.err
