# round-2 batch s: row panels as their own kernel (main product back to 0 spills); A/B stream-tile rows 128 vs 256;
# GPU suite; C5 bench; drop-in + speculative B&B with the low-priority stream
bash tools/ab_bench.sh paper_2510_10891_b200/libhprlp_b200.so tools/ab_rows256.so 3 > gpurun_out/r2s_rows.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r2s_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2s_pytest.log
python bench.py --config C5 --steps 8 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2s_c5.json 2> gpurun_out/r2s_c5.err
