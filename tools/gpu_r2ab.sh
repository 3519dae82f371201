# round-2 batch ab: fused vs split at C5 and C3
for f in 0 1 0 1; do
  HPR_FUSED=$f timeout 600 python bench.py --config C5 --no-e2e --no-cpu-baseline --no-screen --steps 8 > gpurun_out/ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('C5 fused=$f', round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()}, round(d['check_block_us'],1), d['clocks']['sm_mhz'])" >> gpurun_out/r2ab.txt
done
for f in 0 1 0 1; do
  HPR_FUSED=$f timeout 600 python bench.py --config C3 --no-e2e --no-cpu-baseline --no-screen --steps 30 > gpurun_out/ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('C3 fused=$f', round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()}, round(d['check_block_us'],1))" >> gpurun_out/r2ab.txt
done
