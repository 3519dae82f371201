mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_screen.py -m gpu -x -q -k "sizes_and_edges or matches_reference" > gpurun_out/r1k_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r1k_memcheck.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_screen.py -m gpu -x -q -k "matches_reference" > gpurun_out/r1k_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r1k_racecheck.log
timeout 800 python tools/sf_e2e.py --backend gpu --config C1 --time-limit 600 --shutdown-feasible --out gpurun_out/r1k_sf_c1.json > gpurun_out/r1k_sf_c1.log 2>&1; echo "sf rc=$?" >> gpurun_out/r1k_sf_c1.log
echo DONE
