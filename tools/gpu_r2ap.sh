# round-2 batch ap: FP64 record rerun (r2ao saw a 1,830 MHz median clock)
python bench.py > gpurun_out/r2ap_bench.json 2> gpurun_out/r2ap_bench.err
