"""Launch each fused iteration kernel once outside the loop graph so ncu can
capture it in isolation:  ncu -k regex:EpiDual|EpiPrimal ... python tools/profile_kernels.py"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--precision", default="fp64")
ap.add_argument("--reorder", type=int, default=1)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()

import torch  # noqa: E402

from paper_2510_10891_b200 import hprlp, scuc  # noqa: E402
from paper_2510_10891_b200.lp import Precision  # noqa: E402

doc, mon, lpa = scuc.build_config(a.config, device="cuda:0")
eng = hprlp.Engine(lpa.to_lp(), reorder=bool(a.reorder))
eng.solve_raw(hprlp.SolverConfig(tolerance=1e-4, ruiz=False, precision=Precision(a.precision),
                                 max_iterations=0))
t_dual = eng.bench_kernel(0, a.reps)
t_primal = eng.bench_kernel(1, a.reps)
t_at = eng.bench_kernel(2, a.reps)
t_a = eng.bench_kernel(3, a.reps)
torch.cuda.synchronize()
print(f"{os.environ.get('HPR_LIB', 'default')} {os.environ.get('HPR_SPMV', 'pipe')} {a.config} "
      f"{lpa.shape} nnz={lpa.nnz} dual {t_dual*1e6:.1f} us primal {t_primal*1e6:.1f} us "
      f"| plain A {t_a*1e6:.1f} us  plain AT {t_at*1e6:.1f} us")
