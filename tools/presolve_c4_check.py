"""C4 presolve: the native core + native matrix cut against the reference's
own milp_presolve / lp_presolve on the same model (build container only: it
imports the reference).  Prints one JSON line with timings and the identity
verdict (every field of the reduced models and logs, dtypes included)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.append("/root/reference/pkg/src")
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
from scuckit import formulation as F, lp_kernel as K, parse_instance  # noqa: E402
from scuckit import presolve as R  # noqa: E402
from paper_2510_10891_b200 import builder, presolve as P, scuc  # noqa: E402
from paper_2510_10891_b200 import _capi  # noqa: E402
from paper_2510_10891_b200.lp import lazy_csc_matrix  # noqa: E402
from tests.test_presolve import _same  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
_capi.load()                     # library load (and its torch import) outside the clocks
t = time.perf_counter()
doc, mon, lpa = scuc.build_config(cfg)
inst = parse_instance(doc)
vmap = F.VariableMap(inst)
csr = sp.csr_matrix((lpa.data, lpa.indices, lpa.indptr), shape=lpa.shape)
mon = sorted(set(mon))
lp = K.StandardFormLp(matrix=K.SparseMatrix(csr), rhs=lpa.rhs, cost=lpa.cost, lower=lpa.lower,
                      upper=lpa.upper, n_eq=lpa.n_eq, row_tags=builder._row_tags(inst, mon),
                      col_tags=builder._col_tags(inst, vmap))
model = F.MilpModel(lp, vmap.binary_mask.copy(), vmap)
out = {"config": cfg, "shape": list(csr.shape), "nnz": int(csr.nnz),
       "build_s": time.perf_counter() - t}
P._LOG_CLASS = R.ReductionLog
t = time.perf_counter(); ours = P.milp_presolve(model); out["native_milp_s"] = time.perf_counter() - t
lp2 = ours[0].relax()
t = time.perf_counter(); ours_lp = P.lp_presolve(lp2); out["native_lp_s"] = time.perf_counter() - t
t = time.perf_counter(); ref = R.milp_presolve(model); out["ref_milp_s"] = time.perf_counter() - t
t = time.perf_counter(); ref_lp = R.lp_presolve(ref[0].relax()); out["ref_lp_s"] = time.perf_counter() - t
_same(ref, ours)
_same(ref_lp, ours_lp)
out.update(identical=True, bound_changes=len(ref[1].bound_changes),
           removed_rows=len(ref[1].removed_rows))
print(json.dumps(out), flush=True)
