# round-2 batch aj: records with in-iteration kernel timings; standalone vs in-iteration per kernel; GPU suite
python bench.py > gpurun_out/r2aj_bench.json 2> gpurun_out/r2aj_bench.err
python bench.py --precision fp32 --no-screen > gpurun_out/r2aj_fp32.json 2> gpurun_out/r2aj_fp32.err
for p in fp64 fp32; do
  python tools/profile_kernels.py --precision $p --which 5,6,0,1,2,3 --reps 20 > gpurun_out/r2aj_kernels_$p.txt 2>&1
  python tools/profile_kernels.py --precision $p --which 5,6,0,1,2,3 --reps 20 --in-iteration >> gpurun_out/r2aj_kernels_$p.txt 2>&1
done
python -m pytest tests -m gpu -x -q > gpurun_out/r2aj_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2aj_pytest.log
