# round-2 batch ao: final records (FP64 default, FP32), ncu of the final fused pair, launch list, smoke
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2ao_smoke.log 2>&1
python bench.py > gpurun_out/r2ao_bench.json 2> gpurun_out/r2ao_bench.err
python bench.py --precision fp32 --no-screen > gpurun_out/r2ao_fp32.json 2> gpurun_out/r2ao_fp32.err
python tools/profile_kernels.py --which 5,6 --reps 20 > gpurun_out/r2ao_kernels.txt 2>&1
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none --import-source on -c 4 \
    -o gpurun_out/r03_iter_final_fused -f python tools/profile_kernels.py --reps 1 --which 5,6 > gpurun_out/r03_ncu_final_fused.log 2>&1
ncu -i gpurun_out/r03_iter_final_fused.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct > gpurun_out/r03_iter_final_fused_raw.csv 2>&1
HPR_EAGER=1 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r03_launches_final.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-screen > gpurun_out/r03_launches_final_bench.log 2>&1
