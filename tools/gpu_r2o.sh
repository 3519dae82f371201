# round-2 ncu batch o: eager launch list of the timed step at C4; C5 A x~ with row panels (--set full)
HPR_EAGER=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 2500 --csv \
    --log-file gpurun_out/r03_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-screen > gpurun_out/r03_launches_bench.log 2>&1
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none -c 2 \
    -o gpurun_out/r03_iter_c5rp -f python tools/profile_kernels.py --config C5 --reps 1 --which 0,1 > gpurun_out/r03_ncu_c5rp.log 2>&1
ncu -i gpurun_out/r03_iter_c5rp.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,lts__t_sector_hit_rate.pct > gpurun_out/r03_iter_c5rp_raw.csv 2>&1
python tools/traj_probe.py --c4full --out gpurun_out/r2o_traj_full.json > gpurun_out/r2o_traj_full.log 2>&1
