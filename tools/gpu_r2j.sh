# round-2 batch j: row panels for A x~ (A/B at C4 and C5), GPU suite incl. the C4 window (pinned build pool)
for v in 0 1; do HPR_ROWPANELS=$v python bench.py --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2j_c4_rp$v.json 2> gpurun_out/r2j_c4_rp$v.err; done
for v in 0 1; do HPR_ROWPANELS=$v python bench.py --config C5 --steps 8 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2j_c5_rp$v.json 2> gpurun_out/r2j_c5_rp$v.err; done
python -m pytest tests -m gpu -x -q > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2j_pytest.log
python tools/traj_probe.py --c4 --out gpurun_out/r2j_traj.json > gpurun_out/r2j_traj.log 2>&1
