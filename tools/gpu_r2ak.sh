# round-2 batch ak: A/B of the paired dual epilogue (both rows' frow entries in one round trip)
bash tools/ab_bench.sh tools/ab_pair0.so tools/ab_pair1.so 3 > gpurun_out/r2ak_ab64.txt 2>&1
bash tools/ab_bench_fp32.sh tools/ab_pair0.so tools/ab_pair1.so 2 > gpurun_out/r2ak_ab32.txt 2>&1
