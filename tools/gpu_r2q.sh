# round-2 batch q: C1 end-to-end successive fixing with the full drop-in (speculative B&B on)
timeout 1500 python tools/sf_e2e.py --backend gpu --config C1 --time-limit 1200 --shutdown-feasible --out gpurun_out/r2q_sf_c1_gpu.json > gpurun_out/r2q_sf_c1.log 2>&1
