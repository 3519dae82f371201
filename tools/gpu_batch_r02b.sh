# r02: persistent SpMV + deferred long rows — tests, then bench both launch shapes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|FAILED|^E " gpurun_out/pytest_gpu.log | tail -8
for p in 1 0 1; do
  HPR_PERSIST=$p timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 50 > gpurun_out/bench_persist$p.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_persist$p.log').read().strip().splitlines()[-1]);print('persist=$p', round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()}, round(d['check_block_us'],1), round(d['launch_gap_us_per_iteration'],1))"
done
timeout 900 python tools/small_lp_probe.py > gpurun_out/small_lp.log 2>&1; echo small=$?; cat gpurun_out/small_lp.log | tail -4
