"""Launch each kernel of one HPR iteration outside the loop graph, inside an
NVTX range "iter", so ncu can capture them in isolation:

    ncu --nvtx --nvtx-include "iter/" --set full ... python tools/profile_kernels.py --reps 1

Prints the CUDA-event time of every kernel (average over --reps launches).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--precision", default="fp64")
ap.add_argument("--reorder", type=int, default=1)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--which", default="0,1,2,3")
ap.add_argument("--in-iteration", action="store_true",
                help="follow each timed launch by the rest of its iteration (loop cache state)")
a = ap.parse_args()

import torch  # noqa: E402

from paper_2510_10891_b200 import hprlp, scuc  # noqa: E402
from paper_2510_10891_b200.lp import Precision  # noqa: E402

NAMES = {0: "spmv_A", 1: "spmv_AT", 2: "update_primal", 3: "update_dual",
         5: "spmv_AT+primal", 6: "spmv_A+dual"}
doc, mon, lpa = scuc.build_config(a.config)
eng = hprlp.Engine(lpa.to_lp(), reorder=bool(a.reorder))
eng.solve_raw(hprlp.SolverConfig(tolerance=1e-4, ruiz=False, precision=Precision(a.precision),
                                 max_iterations=0))
torch.cuda.synchronize()
out = []
with torch.cuda.nvtx.range("iter"):
    for w in [int(v) for v in a.which.split(",")]:
        out.append(f"{NAMES[w]} {eng.bench_kernel(w, a.reps, in_iteration=a.in_iteration) * 1e6:.1f} us")
torch.cuda.synchronize()
print(f"{os.environ.get('HPR_LIB', 'default')} {a.config} {a.precision} {lpa.shape} "
      f"nnz={lpa.nnz} | " + " | ".join(out))
