# round-2 batch k: row panels (2 rows per warp step) A/B at C4 and C5
for v in 0 1; do HPR_ROWPANELS=$v python tools/profile_kernels.py --reps 20 --which 0 >> gpurun_out/r2k_c4.txt 2>&1; done
for v in 0 1; do HPR_ROWPANELS=$v python tools/profile_kernels.py --config C5 --reps 5 --which 0 >> gpurun_out/r2k_c5.txt 2>&1; done
