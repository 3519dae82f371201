"""Golden warm-started solves of the UNMODIFIED reference (build container
only):  python tests/golden/make_warm_golden.py

B&B node LPs start from the parent's point (milp_bb.py:241-242, start=).  For
6 random LPs of random_lps.npz the reference solves from a perturbed copy of
its own FP64 optimum (seeded noise) at tol 1e-7, FP64 and FP32; the starts and
the results go to tests/golden/warm_starts.npz."""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from scuckit import hprlp  # noqa: E402
from scuckit.lp_kernel import Precision, SparseMatrix, StandardFormLp  # noqa: E402

from tests import golden_io  # noqa: E402

KEYS = ("iterations", "restarts", "objective", "lam", "sigma_final")

if __name__ == "__main__":
    arrays, meta = {}, []
    for i, (lp, _, res) in enumerate(golden_io.random_lps()[:6]):
        rng = np.random.default_rng(100 + i)
        start = [np.asarray(res["fp64"][c]) * (1.0 + 0.1 * rng.standard_normal(len(res["fp64"][c])))
                 + 0.01 * rng.standard_normal(len(res["fp64"][c])) for c in "xyz"]
        for c, v in zip("xyz", start):
            arrays[f"lp{i}_{c}0"] = v
        ref = StandardFormLp(matrix=SparseMatrix(lp.matrix.csr), rhs=lp.rhs, cost=lp.cost,
                             lower=lp.lower, upper=lp.upper, n_eq=lp.n_eq, offset=lp.offset)
        rec = {}
        for prec in ("fp64", "fp32"):
            r = hprlp.solve(ref, hprlp.SolverConfig(tolerance=1e-7 if prec == "fp64" else 1e-5,
                                                    precision=Precision(prec)),
                            start=tuple(start))
            rec[prec] = {k: float(getattr(r, k)) for k in KEYS}
            rec[prec]["status"] = r.status.value
        meta.append(rec)
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "warm_starts.npz"), **arrays)
    print([(m["fp64"]["iterations"], m["fp32"]["iterations"]) for m in meta])
