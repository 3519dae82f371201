# round-2 batch am: committed build vs FP64-only paired dual loads (pp0) vs + paired primal columns (pp1)
for i in 1 2 3; do for L in tools/ab_base.so tools/ab_pp0.so tools/ab_pp1.so; do
  HPR_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-screen --steps 30 > gpurun_out/ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$L'.split('/')[-1], 'fp64', round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()})"
done; done > gpurun_out/r2am_ab64.txt 2>&1
for i in 1 2; do for L in tools/ab_base.so tools/ab_pp0.so tools/ab_pp1.so; do
  HPR_LIB=$L timeout 300 python bench.py --precision fp32 --no-e2e --no-cpu-baseline --no-screen --steps 30 > gpurun_out/ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$L'.split('/')[-1], 'fp32', round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()})"
done; done > gpurun_out/r2am_ab32.txt 2>&1
