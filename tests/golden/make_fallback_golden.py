"""FP32 -> FP64 retry fixture (``hprlp.solve``, hprlp.py:319-329): a 2 x 2 LP
whose lower bound (1e39) is finite in FP64 but overflows to inf in the FP32
work copy (hprlp.py:338-343), so the FP32 iterates lose finiteness, the
reference reports numerical-failure internally and reruns in FP64 with
``fp64_fallback=True``.  Made by the UNMODIFIED reference in the build
container:

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_fallback_golden.py
"""
import json
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import scipy.sparse as sp  # noqa: E402
from scuckit import hprlp, lp_kernel  # noqa: E402

LP = dict(a=[[1.0, 1.0], [1.0, -1.0]], rhs=[1.0, 0.0], cost=[1.0, 2.0],
          lower=[1e39, 0.0], upper=[2e39, 1e3], n_eq=0)


def main():
    lp = lp_kernel.StandardFormLp(matrix=lp_kernel.SparseMatrix(sp.csr_matrix(np.array(LP["a"]))),
                                  rhs=np.array(LP["rhs"]), cost=np.array(LP["cost"]),
                                  lower=np.array(LP["lower"]), upper=np.array(LP["upper"]),
                                  n_eq=LP["n_eq"])
    out = {"lp": LP}
    for tag, prec in (("fp64", lp_kernel.Precision.FP64), ("fp32", lp_kernel.Precision.FP32)):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = hprlp.solve(lp, hprlp.SolverConfig(tolerance=1e-8, precision=prec,
                                                   max_iterations=2000))
        out[tag] = {"status": r.status.value, "iterations": r.iterations,
                    "restarts": r.restarts, "objective": r.objective,
                    "fp64_fallback": bool(r.fp64_fallback),
                    "precision_used": r.precision_used.value, "x": r.x.tolist()}
        print(tag, out[tag])
    with open(os.path.join(HERE, "fallback.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
