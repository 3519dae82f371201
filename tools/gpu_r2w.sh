# round-2 batch w: F^T panel tiles as their own kernel (k_spmv_panels) vs inline; batch depth / occupancy
L0=paper_2510_10891_b200/libhprlp_b200.so
for i in 1 2; do
  for cfg in "$L0 0" "$L0 1" "tools/ab_pu12.so 1" "tools/ab_pu16.so 1"; do set -- $cfg
    HPR_LIB=$1 HPR_PANELKERNEL=$2 timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-screen --steps 30 > gpurun_out/ab.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$1'.split('/')[-1], 'pk=$2', round(d['value'],1), round(d['iteration_us'],1), {k: round(v['us'],1) for k,v in d['kernels'].items()}, round(d['check_block_us'],1))" >> gpurun_out/r2w_c4.txt
  done
done
for cfg in "$L0 0" "$L0 1" "tools/ab_pu12.so 1" "tools/ab_pu16.so 1"; do set -- $cfg
  HPR_LIB=$1 HPR_PANELKERNEL=$2 python tools/profile_kernels.py --config C5 --reps 5 --which 1 >> gpurun_out/r2w_c5.txt 2>&1; echo "  ^ pk=$2" >> gpurun_out/r2w_c5.txt
done
