# round-2 batch ah: C1 end-to-end SF with speculative sibling solves on a default-priority stream
# (the engine's own solves on greatest-priority private streams)
timeout 1500 python tools/sf_e2e.py --backend gpu --config C1 --time-limit 1200 --shutdown-feasible --bb --out gpurun_out/r2ah_sf_c1_spec.json > gpurun_out/r2ah_sf_c1_spec.log 2>&1
