# round-2 batch aa: fused vs split iteration at C4 with the round-2 tiles, FP64 and FP32
for i in 1 2; do for f in 0 1; do for p in fp64 fp32; do
  HPR_FUSED=$f timeout 300 python bench.py --precision $p --no-e2e --no-cpu-baseline --no-screen --steps 30 > gpurun_out/ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('fused=$f $p', round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()}, round(d['check_block_us'],1))" >> gpurun_out/r2aa.txt
done; done; done
