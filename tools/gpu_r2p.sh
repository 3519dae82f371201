# round-2 batch p: speculative B&B tests + drop-in suite; launch list of the timed region (eager, NVTX)
python -m pytest tests/test_dropin_fixing.py -x -q -s > gpurun_out/r2p_dropin.log 2>&1; echo "rc $?" >> gpurun_out/r2p_dropin.log
HPR_EAGER=1 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r03_launches_timed.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-screen > gpurun_out/r03_launches_timed_bench.log 2>&1
