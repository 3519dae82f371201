# round-2 batch x: panel kernel defaults (own kernel from 100M panel entries, 8 CTAs/SM x 16 loads); GPU suite; C5 record
python -m pytest tests -m gpu -x -q > gpurun_out/r2x_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2x_pytest.log
python bench.py --config C5 --steps 10 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2x_c5.json 2> gpurun_out/r2x_c5.err
python tools/profile_kernels.py --config C5 --reps 5 > gpurun_out/r2x_kernels_c5.txt 2>&1
python bench.py --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2x_c4.json 2> gpurun_out/r2x_c4.err
