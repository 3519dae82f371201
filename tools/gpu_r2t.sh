# round-2 batch t: k_spmv_rows occupancy A/B at C5 (16 default vs 8 vs 12 CTAs/SM); C4 bench with rows256 default
for L in paper_2510_10891_b200/libhprlp_b200.so tools/ab_rp8.so tools/ab_rp12.so paper_2510_10891_b200/libhprlp_b200.so; do
  HPR_LIB=$L python tools/profile_kernels.py --config C5 --reps 5 --which 0 >> gpurun_out/r2t_c5.txt 2>&1; done
python bench.py --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2t_c4.json 2> gpurun_out/r2t_c4.err
