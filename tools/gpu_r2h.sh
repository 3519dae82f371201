# round-2 batch h: C5 bench lines (N=1 single engine; partitioned mode at world size 1), drop-in tests
python bench.py --config C5 --steps 10 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2h_c5.json 2> gpurun_out/r2h_c5.err
python bench.py --config C5 --mode partitioned --steps 10 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2h_c5_part.json 2> gpurun_out/r2h_c5_part.err
python -m pytest tests/test_dropin_fixing.py -x -q -s > gpurun_out/r2h_dropin.log 2>&1; echo "rc $?" >> gpurun_out/r2h_dropin.log
