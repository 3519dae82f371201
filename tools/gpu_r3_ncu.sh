# round-2 ncu batch: the four iteration kernels at C4 (--set full), C5 products, eager launch list
python tools/profile_kernels.py --reps 20 > gpurun_out/r03_kernels_c4.txt 2>&1
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none --import-source on -c 4 \
    -o gpurun_out/r03_iter -f python tools/profile_kernels.py --reps 1 > gpurun_out/r03_ncu_iter.log 2>&1
ncu -i gpurun_out/r03_iter.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,smsp__average_warp_latency_issue_stalled_long_scoreboard,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct > gpurun_out/r03_iter_raw.csv 2>&1
python tools/profile_kernels.py --config C5 --reps 5 > gpurun_out/r03_kernels_c5.txt 2>&1
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none -c 2 \
    -o gpurun_out/r03_iter_c5 -f python tools/profile_kernels.py --config C5 --reps 1 --which 0,1 > gpurun_out/r03_ncu_c5.log 2>&1
ncu -i gpurun_out/r03_iter_c5.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,lts__t_sector_hit_rate.pct > gpurun_out/r03_iter_c5_raw.csv 2>&1
HPR_EAGER=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r03_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r03_launches_bench.log 2>&1
