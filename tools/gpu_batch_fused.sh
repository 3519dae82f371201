mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|FAILED|^E " gpurun_out/pytest_gpu.log | tail -8
for v in "HPR_FUSED=0" "HPR_FUSED=1"; do
  echo "== $v"; env $v timeout 600 python tools/small_lp_probe.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['tol'], d['iterations'], round(d['us_per_it'],2), round(d['create_s'],3), d['status'])"
done
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_c4.log').read().strip().splitlines()[-1]);print('C4', round(d['value'],1), round(d['iteration_us'],1))"
for cfg in C3; do HPR_FUSED=1 timeout 300 python bench.py --config $cfg --triples 2000 --no-e2e --no-cpu-baseline > gpurun_out/bench_$cfg.f1.log 2>&1; HPR_FUSED=0 timeout 300 python bench.py --config $cfg --triples 2000 --no-e2e --no-cpu-baseline > gpurun_out/bench_$cfg.f0.log 2>&1; for f in 0 1; do python -c "import json;d=json.loads(open('gpurun_out/bench_$cfg.f$f.log').read().strip().splitlines()[-1]);print('$cfg fused=$f', round(d['value'],1), round(d['iteration_us'],1), d['config']['device_layout'])"; done; done
