# round-2 batch af: records with the fused default + scratch-pool retention; ncu of the fused dual product
python bench.py > gpurun_out/r2af_bench.json 2> gpurun_out/r2af_bench.err
python bench.py --precision fp32 --no-screen > gpurun_out/r2af_fp32.json 2> gpurun_out/r2af_fp32.err
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none --import-source on -c 1 \
    -o gpurun_out/r03_iter_fused_dual -f python tools/profile_kernels.py --reps 1 --which 6 > gpurun_out/r03_ncu_fused_dual.log 2>&1
ncu -i gpurun_out/r03_iter_fused_dual.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct > gpurun_out/r03_iter_fused_dual_raw.csv 2>&1
