# SF end-to-end on C2, B200 backend (fused small-LP iteration + native presolve)
mkdir -p gpurun_out
timeout 1300 python tools/sf_e2e.py --backend gpu --config C2 --time-limit 1200 --shutdown-feasible --out gpurun_out/sf_C2_gpu_b.json > gpurun_out/sf_C2_gpu_b.log 2>&1; echo sf_C2_gpu=$?
tail -c 600 gpurun_out/sf_C2_gpu_b.log
