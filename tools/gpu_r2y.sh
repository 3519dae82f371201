# round-2 batch y: column-sharded primal update (reduce-scatter + all-gather) in partitioned mode
python -m pytest tests/test_gpu_parity.py -x -q -k partitioned > gpurun_out/r2y_part.log 2>&1; echo "rc $?" >> gpurun_out/r2y_part.log
python -m pytest tests -m gpu -x -q > gpurun_out/r2y_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2y_pytest.log
python bench.py --config C5 --mode partitioned --steps 10 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2y_c5_part.json 2> gpurun_out/r2y_c5_part.err
python bench.py --mode partitioned --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2y_c4_part.json 2> gpurun_out/r2y_c4_part.err
