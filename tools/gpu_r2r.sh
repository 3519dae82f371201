# round-2 batch r: A/B of stream-tile row cap 128 vs 256, and check-grid 4736 vs 1184 slots
bash tools/ab_bench.sh paper_2510_10891_b200/libhprlp_b200.so tools/ab_rows256.so 3 > gpurun_out/r2r_rows.txt 2>&1
bash tools/ab_bench.sh paper_2510_10891_b200/libhprlp_b200.so tools/ab_grid1184.so 3 > gpurun_out/r2r_grid.txt 2>&1
