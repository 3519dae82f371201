# round-2 batch a: GPU suite after the host sigma update / device scope changes,
# trajectory diffs vs the committed reference records, a short bench
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2a_pytest.log
python tools/traj_probe.py --out gpurun_out/r2a_traj.json > gpurun_out/r2a_traj.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
