# round-2 batch al: A/B of pairing the dual epilogue's y / rhs / anchor loads too (ab_pl1) against the committed build
bash tools/ab_bench.sh tools/ab_base.so tools/ab_pl1.so 3 > gpurun_out/r2al_ab64.txt 2>&1
bash tools/ab_bench_fp32.sh tools/ab_base.so tools/ab_pl1.so 2 > gpurun_out/r2al_ab32.txt 2>&1
