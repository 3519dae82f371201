"""Reference trajectory on the exact C4 bench LP (the BASELINE headline config:
13,659-bus / 4,092-unit / 36-period SCUC relaxation + 1,000 base flow triples,
1,769,780 x 1,670,220, 44.3M nnz), made by running the UNMODIFIED reference
``scuckit.hprlp.solve`` (/root/reference/pkg/src, hprlp.py:319-455) in the build
container:

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_c4_golden.py window
    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_c4_golden.py full fp64

``window`` writes tests/golden/c4_window.json: the first 2,048 iterations
(128 checks) in FP64 and FP32 with ``SolverConfig(tolerance=1e-4, ruiz=False,
log_residuals=True, max_iterations=2048)`` -- the driver's solver setting
(driver.py:54, :61-65) -- with lambda, sigma0, b/c scales, every residual-log
row, the restart list (check iteration, kind, sigma before/after), the
iteration-limit result's objective and KKT fields, and a fixed sample of the
returned best triple.  ``full <prec>`` writes c4_full_<prec>.json: the same
record for the run to tolerance (~7 h in FP64 on one core).

The LP digest is recorded; scuc.build_config solves its PTDF rows under the
pinned BLAS pool, so the B200 box rebuilds the identical LP and
tests/test_gpu_parity.py::test_c4_window_against_reference asserts the digest
before comparing.  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from scuckit import hprlp, lp_kernel  # noqa: E402

from paper_2510_10891_b200 import scuc  # noqa: E402
from tests import golden_io  # noqa: E402

SAMPLE = 64


def ref_lp(lpa):
    import scipy.sparse as sp
    mat = lp_kernel.SparseMatrix(sp.csr_matrix((lpa.data, lpa.indices, lpa.indptr),
                                               shape=lpa.shape))
    return lp_kernel.StandardFormLp(matrix=mat, rhs=lpa.rhs, cost=lpa.cost, lower=lpa.lower,
                                    upper=lpa.upper, n_eq=lpa.n_eq, offset=lpa.offset)


def sample_idx(n, seed):
    return np.sort(np.random.default_rng(seed).choice(n, size=min(SAMPLE, n), replace=False))


def record(lp, lpa, cfg, r):
    maps = hprlp._ScaleMaps(lp, cfg)
    log = r.residual_log
    n, m = lpa.shape[1], lpa.shape[0]
    ix, iy = sample_idx(n, 11), sample_idx(m, 12)
    out = {
        "status": r.status.value, "iterations": r.iterations, "restarts": r.restarts,
        "objective": r.objective, "lam": r.lam, "sigma_final": r.sigma_final,
        "sigma0": log[0]["sigma"] if log else None,
        "b_scale": maps.b_scale, "c_scale": maps.c_scale,
        "kkt": {k: float(getattr(r.kkt, k)) for k in (
            "primal", "box", "dual", "rel_primal", "rel_box", "rel_dual",
            "primal_objective", "dual_objective", "gap", "rel_gap")},
        "log": [[e["iteration"], e["epoch"], e["rel_primal"], e["rel_dual"], e["rel_box"],
                 e["rel_gap"], e["sigma"]] for e in log],
        "restart_list": [dict(zip(("iteration", "kind", "sigma", "sigma_after"), t))
                         for t in golden_io.restart_list(
                             [[e[k] for k in golden_io.LOG_COLS] for e in log],
                             cfg.restart_beta, cfg.restart_stall)],
        "sample": {"x_idx": ix.tolist(), "x": r.x[ix].tolist(),
                   "y_idx": iy.tolist(), "y": r.y[iy].tolist(), "z": r.z[ix].tolist(),
                   "x_norm": float(np.linalg.norm(r.x)), "y_norm": float(np.linalg.norm(r.y)),
                   "z_norm": float(np.linalg.norm(r.z))},
        "solve_time_s": r.solve_time,
    }
    return out


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "window"
    t = time.perf_counter()
    doc, mon, lpa = scuc.build_config("C4")
    print("built", lpa.shape, lpa.nnz, lpa.digest(), round(time.perf_counter() - t, 1), flush=True)
    lp = ref_lp(lpa)
    head = {"config": "C4", "n_triples": 1000, "digest": lpa.digest(), "shape": list(lpa.shape),
            "nnz": lpa.nnz, "n_eq": lpa.n_eq}
    if mode == "window":
        out = dict(head, max_iterations=2048)
        for tag, prec in (("fp64", lp_kernel.Precision.FP64), ("fp32", lp_kernel.Precision.FP32)):
            cfg = hprlp.SolverConfig(tolerance=1e-4, ruiz=False, precision=prec,
                                     log_residuals=True, max_iterations=2048)
            r = hprlp.solve(lp, cfg)
            out[tag] = record(lp, lpa, cfg, r)
            print(tag, r.status.value, r.iterations, r.restarts, r.objective, r.solve_time,
                  flush=True)
        path = os.path.join(HERE, "c4_window.json")
    else:
        tag = sys.argv[2]
        prec = lp_kernel.Precision.FP64 if tag == "fp64" else lp_kernel.Precision.FP32
        cfg = hprlp.SolverConfig(tolerance=1e-4, ruiz=False, precision=prec, log_residuals=True)
        r = hprlp.solve(lp, cfg)
        out = dict(head, **{tag: record(lp, lpa, cfg, r)})
        print(tag, r.status.value, r.iterations, r.restarts, r.objective, r.solve_time,
              flush=True)
        path = os.path.join(HERE, f"c4_full_{tag}.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print("wrote", path)


if __name__ == "__main__":
    main()
