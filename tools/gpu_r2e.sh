# round-2 batch e: C4 window vs the reference (new golden), C5 build + window
python tools/traj_probe.py --c4 --out gpurun_out/r2e_traj.json > gpurun_out/r2e_traj.log 2>&1
python -m pytest tests/test_gpu_trajectories.py -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2e_pytest.log
timeout 1500 python tools/c5_probe.py --iters 256 > gpurun_out/r2e_c5.log 2>&1
