# round-2 batch ai: C1 end-to-end SF on the same build without speculation (the r2ah comparison)
timeout 1500 python tools/sf_e2e.py --backend gpu --config C1 --time-limit 1200 --shutdown-feasible --out gpurun_out/r2ai_sf_c1.json > gpurun_out/r2ai_sf_c1.log 2>&1
