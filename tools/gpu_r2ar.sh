# round-2 batch ar: the engine against the reference's full C4 FP64 run (c4_full_fp64.json)
python tools/traj_probe.py --c4full --out gpurun_out/r2ar_traj_c4full.json > gpurun_out/r2ar_traj.log 2>&1
python -m pytest tests/test_gpu_trajectories.py -m gpu -q -k "c4_full" > gpurun_out/r2ar_pytest_c4full.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2ar_pytest_c4full.log
