import time, json, numpy as np, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2510_10891_b200 import scuc, hprlp
from paper_2510_10891_b200.lp import Precision
t=time.time(); doc, mon, lpa = scuc.build_config("C1"); print("build", time.time()-t, lpa.shape, lpa.nnz, lpa.digest())
lp = lpa.to_lp()
for prec in ["fp64", "fp32"]:
    for rep in range(2):
        t=time.time(); r = hprlp.solve(lp, hprlp.SolverConfig(tolerance=1e-4, ruiz=False, precision=Precision(prec), log_residuals=True)); dt=time.time()-t
        print(prec, r.status.value, r.iterations, r.restarts, r.objective, r.lam, r.sigma_final, f"wall {dt:.3f}s", r.device_stats, f"it/s(loop) {r.iterations/max(r.device_stats['loop_seconds'],1e-9):.0f}")
