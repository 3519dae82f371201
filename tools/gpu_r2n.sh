# round-2 batch n: end-to-end successive fixing at C4 with the whole drop-in installed
# (LP solves, presolve, screen, model builder); 1,200 s driver time limit
timeout 1700 python tools/sf_e2e.py --backend gpu --config C4 --time-limit 1200 --shutdown-feasible --out gpurun_out/r2n_sf_c4_gpu.json > gpurun_out/r2n_sf_c4.log 2>&1
