# round-2 batch d: column-per-thread flow panels (A^T y); GPU suite, trajectories, bench, kernel times
python -m pytest tests -m gpu -x -q -k "not c4_window" > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2d_pytest.log
python tools/traj_probe.py --out gpurun_out/r2d_traj.json > gpurun_out/r2d_traj.log 2>&1
python bench.py --steps 30 --warmup 3 --no-e2e > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
