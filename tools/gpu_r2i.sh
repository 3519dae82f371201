# round-2 batch i: halt-flag queued partitioned loop, panels in partitioned mode; full GPU suite; C4 bench; C5 partitioned
python -m pytest tests -m gpu -x -q -k "not c4_window" > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2i_pytest.log
python bench.py --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
python bench.py --config C5 --mode partitioned --steps 10 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2i_c5_part.json 2> gpurun_out/r2i_c5_part.err
