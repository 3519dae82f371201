# round-2 batch b: dense flow-block product probe; trajectory diffs (row-relative metric)
./tools/flow_probe.bin > gpurun_out/r2b_flow.log 2>&1
python tools/traj_probe.py --out gpurun_out/r2b_traj.json > gpurun_out/r2b_traj.log 2>&1
