# round-2 batch ac: fused iteration as the default up to C4; records + ncu of the fused pair; GPU suite
python -m pytest tests -m gpu -x -q > gpurun_out/r2ac_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2ac_pytest.log
python bench.py > gpurun_out/r2ac_bench.json 2> gpurun_out/r2ac_bench.err
python bench.py --precision fp32 --no-screen > gpurun_out/r2ac_fp32.json 2> gpurun_out/r2ac_fp32.err
python tools/profile_kernels.py --reps 20 --which 5,6 > gpurun_out/r2ac_kernels_fused.txt 2>&1
ncu --nvtx --nvtx-include "iter/" --set full --clock-control none --import-source on -c 2 \
    -o gpurun_out/r03_iter_fused -f python tools/profile_kernels.py --reps 1 --which 5,6 > gpurun_out/r03_ncu_fused.log 2>&1
ncu -i gpurun_out/r03_iter_fused.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct > gpurun_out/r03_iter_fused_raw.csv 2>&1
HPR_EAGER=1 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r03_launches_fused.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-screen > gpurun_out/r03_launches_fused_bench.log 2>&1
