# round-2 batch g: PDL determinism diagnostics on C2 (HPR_PDL bit 0: products, bit 1: updates)
python - > gpurun_out/r2g_summary.txt 2>&1 <<'PY'
import os, subprocess, sys
code = """
import hashlib, numpy as np
from paper_2510_10891_b200 import hprlp, scuc
doc, mon, lpa = scuc.build_config('C2', n_triples=500)
lp = lpa.to_lp()
for it in (16, 32, 160, 3000):
    r = hprlp.solve(lp, hprlp.SolverConfig(tolerance=1e-4, ruiz=False, max_iterations=it))
    h = hashlib.sha256(); [h.update(np.ascontiguousarray(v).tobytes()) for v in (r.x, r.y, r.z)]
    print(it, h.hexdigest()[:16], r.restarts, end=' | ')
print()
"""
for env in ({"HPR_PDL": "0"}, {"HPR_PDL": "1"}, {"HPR_PDL": "2"}, {"HPR_PDL": "3"},
            {"HPR_PDL": "1", "HPR_FUSED": "0"}, {"HPR_PDL": "2", "HPR_FUSED": "0"}):
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True)
    print(env, out.stdout.strip(), out.stderr[-300:])
PY
