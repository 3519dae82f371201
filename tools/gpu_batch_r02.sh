set -x
mkdir -p gpurun_out
HPR_PDL=1 timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_pdl.log 2>&1; echo pytest_pdl=$?
grep -E "passed|failed|FAILED|^E " gpurun_out/pytest_pdl.log | tail -8
for pdl in 0 1 0 1; do HPR_PDL=$pdl timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 50 > gpurun_out/bench_pdl$pdl.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_pdl$pdl.log').read().strip().splitlines()[-1]);print('pdl=$pdl', d['value'], d['iteration_us'], d['launch_gap_us_per_iteration'], d['check_block_us'])"; done
timeout 1000 python tools/sf_e2e.py --backend cpu --config C2 --time-limit 900 --out gpurun_out/sf_c2_cpu.json > gpurun_out/sf_c2_cpu.log 2>&1 &
CPID=$!
timeout 1000 python tools/sf_e2e.py --backend gpu --config C2 --time-limit 900 --out gpurun_out/sf_c2_gpu.json > gpurun_out/sf_c2_gpu.log 2>&1; echo sfgpu=$?
tail -c 800 gpurun_out/sf_c2_gpu.log
wait $CPID; echo sfcpu=$?
tail -c 800 gpurun_out/sf_c2_cpu.log
