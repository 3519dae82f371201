# A/B of two builds of the engine on the same box, FP32 work precision:
# bash tools/ab_bench_fp32.sh <libA.so> <libB.so> [rounds]
A=$1; B=$2; R=${3:-2}
for i in $(seq $R); do
  for L in $A $B; do
    HPR_LIB=$L timeout 300 python bench.py --precision fp32 --no-e2e --no-cpu-baseline --no-screen --steps 30 > gpurun_out/ab.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$L'.split('/')[-1], round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()})"
  done
done
