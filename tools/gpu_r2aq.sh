# round-2 batch aq: stream tiles of up to 384 rows (three rows per thread) against 256
bash tools/ab_bench.sh tools/ab_rows256.so tools/ab_rows384.so 3 > gpurun_out/r2aq_ab64.txt 2>&1
bash tools/ab_bench_fp32.sh tools/ab_rows256.so tools/ab_rows384.so 2 > gpurun_out/r2aq_ab32.txt 2>&1
