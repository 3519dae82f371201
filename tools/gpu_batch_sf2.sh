# SF end-to-end, B200 backend only (the CPU reference run is unchanged; profiles/r02_sf_C1_cpu.json)
mkdir -p gpurun_out
timeout 1300 python tools/sf_e2e.py --backend gpu --config C1 --time-limit 1200 --shutdown-feasible --out gpurun_out/sf_C1_gpu_b.json > gpurun_out/sf_C1_gpu_b.log 2>&1; echo sf_C1_gpu=$?
tail -c 600 gpurun_out/sf_C1_gpu_b.log
