set -e
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/profile_kernels.py --reps 20 > gpurun_out/pk_plain.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "iter/" --set full --clock-control none --import-source on -c 8 -o gpurun_out/r02e_iter -f python tools/profile_kernels.py --reps 1 > gpurun_out/ncu_e.log 2>&1
echo DONE
