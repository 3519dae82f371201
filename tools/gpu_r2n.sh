# round-2 batch n: end-to-end successive fixing with the whole drop-in installed
# (LP solves, presolve, screen, model builder); C4 (until the driver stops), C2, C1
timeout 1700 python tools/sf_e2e.py --backend gpu --config C4 --time-limit 1200 --shutdown-feasible --out gpurun_out/r2n_sf_c4_gpu.json > gpurun_out/r2n_sf_c4.log 2>&1
timeout 1300 python tools/sf_e2e.py --backend gpu --config C2 --time-limit 1200 --shutdown-feasible --out gpurun_out/r2n_sf_c2_gpu.json > gpurun_out/r2n_sf_c2.log 2>&1
