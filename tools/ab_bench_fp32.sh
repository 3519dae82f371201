for i in 1 2; do for L in paper_2510_10891_b200/libhprlp_b200_base.so paper_2510_10891_b200/libhprlp_b200.so; do
  HPR_LIB=$L timeout 300 python bench.py --precision fp32 --no-e2e --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$L'.split('/')[-1], round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()})"
done; done
