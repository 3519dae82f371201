# round-2 batch ag: the small-LP regime (C1) — warm kernel times and an ncu capture of the fused pair
python tools/profile_kernels.py --config C1 --which 5,6,0,1,2,3 --reps 50 > gpurun_out/r2ag_c1_kernels.txt 2>&1
python tools/small_lp_probe.py > gpurun_out/r2ag_small_lp.txt 2>&1
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none --import-source on -c 4 \
    -o gpurun_out/r03_iter_c1 -f python tools/profile_kernels.py --config C1 --reps 1 --which 5,6 > gpurun_out/r03_ncu_c1.log 2>&1
ncu -i gpurun_out/r03_iter_c1.ncu-rep --page details --csv > gpurun_out/r03_iter_c1_details.csv 2>&1
