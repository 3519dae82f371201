# round-2 batch f: programmatic dependent launch A/B at C4 (bench, no e2e legs), then bit-identity
for v in 0 1 0 1; do HPR_PDL=$v python bench.py --steps 30 --warmup 3 --no-e2e --no-screen --no-cpu-baseline > gpurun_out/r2f_pdl$v.json 2> gpurun_out/r2f_pdl$v.err; python -c "
import json; b=json.load(open('gpurun_out/r2f_pdl$v.json')); print('PDL=$v', round(b['value'],1), round(b['iteration_us'],2), round(b['launch_gap_us_per_iteration'],2), {k:round(x['us'],1) for k,x in b['kernels'].items()})" >> gpurun_out/r2f_summary.txt; done
python - >> gpurun_out/r2f_summary.txt 2>&1 <<'PY'
import os, subprocess, sys
code = """
import hashlib, numpy as np
from paper_2510_10891_b200 import hprlp, scuc
doc, mon, lpa = scuc.build_config('C2', n_triples=500)
r = hprlp.solve(lpa.to_lp(), hprlp.SolverConfig(tolerance=1e-4, ruiz=False, max_iterations=3000))
h = hashlib.sha256(); [h.update(np.ascontiguousarray(v).tobytes()) for v in (r.x, r.y, r.z)]
print(h.hexdigest(), r.iterations)
"""
for v in ("0", "1"):
    for f in ("0", "1"):
        env = dict(os.environ, HPR_PDL=v, HPR_FUSED=f)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print("digest PDL", v, "FUSED", f, out.stdout.strip(), out.stderr[-300:])
PY
