# round-2 batch u: row panels (own kernel, 16 CTAs/SM) on/off at C4 and C3; GPU suite with the new defaults
for v in 0 1 0 1; do HPR_ROWPANELS=$v python tools/profile_kernels.py --reps 20 --which 0 >> gpurun_out/r2u_c4.txt 2>&1; done
for v in 0 1; do HPR_ROWPANELS=$v python tools/profile_kernels.py --config C3 --reps 20 --which 0 >> gpurun_out/r2u_c3.txt 2>&1; done
HPR_ROWPANELS=1 python bench.py --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2u_c4_rp1.json 2> gpurun_out/r2u_c4_rp1.err
python -m pytest tests -m gpu -x -q > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2u_pytest.log
