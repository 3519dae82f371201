# round-2 batch v: records with the round-2 defaults (rows256 stream tiles, row kernel at 16 CTAs/SM, check grid 148x8)
python bench.py > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err
python bench.py --config C5 --steps 10 --warmup 3 --no-screen --no-cpu-baseline > gpurun_out/r2v_c5.json 2> gpurun_out/r2v_c5.err
python bench.py --precision fp32 --no-screen > gpurun_out/r2v_fp32.json 2> gpurun_out/r2v_fp32.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2v_ref.json 2> gpurun_out/r2v_ref.err
python tools/profile_kernels.py --config C5 --reps 5 > gpurun_out/r2v_kernels_c5.txt 2>&1
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none -c 3 \
    -o gpurun_out/r03_iter_c5final -f python tools/profile_kernels.py --config C5 --reps 1 --which 0 > gpurun_out/r03_ncu_c5final.log 2>&1
ncu -i gpurun_out/r03_iter_c5final.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,lts__t_sector_hit_rate.pct > gpurun_out/r03_iter_c5final_raw.csv 2>&1
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none --import-source on -c 4 \
    -o gpurun_out/r03_iter_final -f python tools/profile_kernels.py --reps 1 > gpurun_out/r03_ncu_final.log 2>&1
ncu -i gpurun_out/r03_iter_final.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct > gpurun_out/r03_iter_final_raw.csv 2>&1
