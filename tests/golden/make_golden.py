"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference (``scuckit`` from /root/reference/pkg/src) in the build container.

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py [--c1]

Outputs (small, committed):
  kat.json            SPEC known-answer tests run
                      through scuckit.hpr_iterate / kkt_residual / power_method
  random_lps.npz      24 random bounded-feasible LPs (SPEC acceptance #1 shape:
                      <=40 vars, <=30 rows, some infinite bounds) with the
                      reference solve at tol 1e-8 (FP64) and 1e-6 (FP32), and
                      the HiGHS objective (scuckit.lp_backends simplex oracle)
  scuc_small.npz      a 30-bus / 12-unit / 8-period SCUC relaxation (all base
                      flow rows) with reference solves and residual logs
  c1_trajectory.json  (--c1) digest of the C1 LP built by
                      paper_2510_10891_b200.scuc + the reference FP64/FP32
                      trajectory at tol 1e-4 (lambda, restarts, sigma, final
                      iteration, objective, per-check residual log)
The /root/reference tree is read here only; nothing on the GPU box reads it.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from scuckit import hprlp, lp_backends, lp_kernel  # noqa: E402

from paper_2510_10891_b200 import scuc  # noqa: E402

RESULT_KEYS = ("iterations", "restarts", "objective", "lam", "sigma_final")


def ref_lp(indptr, indices, data, shape, rhs, cost, lower, upper, n_eq, offset=0.0):
    import scipy.sparse as sp
    mat = lp_kernel.SparseMatrix(sp.csr_matrix((data, indices, indptr), shape=shape))
    return lp_kernel.StandardFormLp(matrix=mat, rhs=np.asarray(rhs, float),
                                    cost=np.asarray(cost, float), lower=np.asarray(lower, float),
                                    upper=np.asarray(upper, float), n_eq=int(n_eq),
                                    offset=float(offset))


def random_lp(rng, inf_bounds=True):
    """Bounded-feasible random LP: primal point inside the box and a dual
    point with sign-consistent reduced costs guarantee an optimum."""
    n = int(rng.integers(5, 41))
    m = int(rng.integers(3, 31))
    n_eq = int(rng.integers(0, m // 3 + 1))
    dens = rng.uniform(0.15, 0.5)
    a = rng.standard_normal((m, n)) * (rng.uniform(size=(m, n)) < dens)
    for i in range(m):                      # no empty rows
        if not a[i].any():
            a[i, rng.integers(0, n)] = rng.standard_normal()
    lower = rng.uniform(-5, 0, n)
    upper = lower + rng.uniform(1, 10, n)
    if inf_bounds:
        k = rng.uniform(size=n)
        upper[k < 0.15] = np.inf
        lower[(k >= 0.15) & (k < 0.25)] = -np.inf
    xf = np.where(np.isfinite(lower), lower, upper - 1.0) + 0.0
    xf = np.where(np.isfinite(lower) & np.isfinite(upper),
                  lower + rng.uniform(0.1, 0.9, n) * (upper - lower), xf)
    xf = np.where(np.isfinite(lower) & ~np.isfinite(upper), lower + rng.uniform(0, 3, n), xf)
    ax = a @ xf
    rhs = ax.copy()
    rhs[n_eq:] -= rng.uniform(0, 2, m - n_eq) * (rng.uniform(size=m - n_eq) < 0.6)
    y = rng.standard_normal(m)
    y[n_eq:] = np.abs(y[n_eq:])
    z = rng.standard_normal(n)
    z = np.where(~np.isfinite(upper), np.abs(z), z)
    z = np.where(~np.isfinite(lower), -np.abs(z), z)
    cost = a.T @ y + z
    import scipy.sparse as sp
    csr = sp.csr_matrix(a)
    csr.sort_indices()
    return dict(indptr=csr.indptr.astype(np.int32), indices=csr.indices.astype(np.int32),
                data=csr.data.astype(np.float64), shape=np.array([m, n]), rhs=rhs, cost=cost,
                lower=lower, upper=upper, n_eq=n_eq)


def res_dict(r):
    d = {k: (float(getattr(r, k)) if k != "iterations" and k != "restarts" else int(getattr(r, k)))
         for k in RESULT_KEYS}
    d["status"] = r.status.value
    d["kkt"] = {k: float(getattr(r.kkt, k)) for k in r.kkt.__dataclass_fields__}
    return d


def make_kat():
    out = {}
    one = ref_lp(np.array([0, 1]), np.array([0]), np.array([1.0]), (1, 1), [1.0], [1.0],
                 [0.0], [2.0], 0)
    st = hprlp.HprState.from_point([1.0], [1.0], [0.0], sigma=1.0, lam=1.0)
    hprlp.hpr_iterate(st, one)
    out["fixed_point_after"] = [float(st.x[0]), float(st.y[0]), float(st.z[0])]
    r = hprlp.kkt_residual(np.array([1.0]), np.array([1.0]), np.array([0.0]), one)
    out["fixed_point_kkt"] = [r.primal, r.box, r.dual]
    st = hprlp.HprState.from_point([0.0], [0.0], [0.0], sigma=1.0, lam=1.0)
    hprlp.hpr_iterate(st, one)
    out["from_zero_bar"] = [float(st.bar_x[0]), float(st.bar_y[0]), float(st.bar_z[0])]
    out["from_zero_next"] = [float(st.x[0]), float(st.y[0]), float(st.z[0])]
    r = hprlp.kkt_residual(np.array([0.5]), np.array([0.0]), np.array([0.0]), one)
    out["primal_residual_x05"] = r.primal
    eye = lp_kernel.SparseMatrix(np.eye(3))
    out["power_identity"] = lp_kernel.power_method(eye)
    out["power_diag21"] = lp_kernel.power_method(lp_kernel.SparseMatrix(np.diag([2.0, 1.0])))
    out["power_identity_solve_inflation"] = lp_kernel.power_method(eye, inflation=1.01)
    res = hprlp.solve(one, hprlp.SolverConfig(tolerance=1e-8))
    out["one_d_solve"] = res_dict(res) | {"x": res.x.tolist(), "y": res.y.tolist(),
                                         "z": res.z.tolist()}
    a = np.array([[1.0, 2.0], [0.0, 3.0]])
    out["matvec_example"] = (a @ np.array([1.0, 1.0])).tolist()
    with open(os.path.join(HERE, "kat.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("kat.json", out["from_zero_bar"], out["power_identity"], out["power_diag21"])


def solve_record(lp, **cfg):
    r = hprlp.solve(lp, hprlp.SolverConfig(**cfg))
    return r


def make_random():
    rng = np.random.default_rng(20251018)
    arrays = {}
    meta = []
    for i in range(24):
        d = random_lp(rng, inf_bounds=(i % 3 != 0))
        lp = ref_lp(**d)
        hi = lp_backends.solve_lp_simplex(lp)
        rec = {"highs_objective": float(hi.objective), "highs_ok": bool(hi.converged)}
        for tag, cfg in (("fp64", dict(tolerance=1e-8)),
                         ("fp32", dict(tolerance=1e-6, precision=lp_kernel.Precision.FP32)),
                         ("fp64_noruiz_log", dict(tolerance=1e-6, ruiz=False, log_residuals=True))):
            r = solve_record(lp, **cfg)
            rec[tag] = res_dict(r)
            arrays[f"lp{i}_{tag}_x"] = r.x
            arrays[f"lp{i}_{tag}_y"] = r.y
            arrays[f"lp{i}_{tag}_z"] = r.z
            if r.residual_log:
                arrays[f"lp{i}_{tag}_log"] = np.array(
                    [[e["iteration"], e["epoch"], e["rel_primal"], e["rel_dual"], e["rel_box"],
                      e["rel_gap"], e["sigma"]] for e in r.residual_log])
        for k, v in d.items():
            arrays[f"lp{i}_{k}"] = np.asarray(v)
        meta.append(rec)
        print(i, d["shape"], rec["fp64"]["status"], rec["fp64"]["iterations"],
              rec["fp64"]["objective"], rec["highs_objective"])
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "random_lps.npz"), **arrays)


def make_scuc_small():
    doc = scuc.generate_instance(30, 12, 45, 8, seed=3)
    lpa = scuc.build_relaxation(doc, scuc.all_base_triples(doc))
    lp = ref_lp(lpa.indptr, lpa.indices, lpa.data, lpa.shape, lpa.rhs, lpa.cost,
                lpa.lower, lpa.upper, lpa.n_eq)
    arrays = dict(indptr=lpa.indptr, indices=lpa.indices, data=lpa.data,
                  shape=np.array(lpa.shape), rhs=lpa.rhs, cost=lpa.cost, lower=lpa.lower,
                  upper=lpa.upper, n_eq=np.array(lpa.n_eq))
    meta = {"digest": lpa.digest()}
    for tag, cfg in (("fp64_1e4", dict(tolerance=1e-4, ruiz=False, log_residuals=True)),
                     ("fp64_1e6_ruiz", dict(tolerance=1e-6, ruiz=True, log_residuals=True,
                                            max_iterations=20000)),
                     ("fp32_1e4", dict(tolerance=1e-4, ruiz=False, log_residuals=True,
                                       precision=lp_kernel.Precision.FP32))):
        r = solve_record(lp, **cfg)
        meta[tag] = res_dict(r)
        arrays[f"{tag}_x"], arrays[f"{tag}_y"], arrays[f"{tag}_z"] = r.x, r.y, r.z
        arrays[f"{tag}_log"] = np.array(
            [[e["iteration"], e["epoch"], e["rel_primal"], e["rel_dual"], e["rel_box"],
              e["rel_gap"], e["sigma"]] for e in r.residual_log])
        print("scuc_small", tag, meta[tag]["status"], meta[tag]["iterations"],
              meta[tag]["restarts"], meta[tag]["objective"])
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "scuc_small.npz"), **arrays)


def make_c1():
    doc, mon, lpa = scuc.build_config("C1")
    lp = ref_lp(lpa.indptr, lpa.indices, lpa.data, lpa.shape, lpa.rhs, lpa.cost,
                lpa.lower, lpa.upper, lpa.n_eq)
    out = {"digest": lpa.digest(), "shape": list(lpa.shape), "nnz": lpa.nnz}
    for tag, prec in (("fp64", lp_kernel.Precision.FP64), ("fp32", lp_kernel.Precision.FP32)):
        r = solve_record(lp, tolerance=1e-4, ruiz=False, precision=prec, log_residuals=True)
        log = r.residual_log
        restarts = [log[i]["iteration"] for i in range(1, len(log))
                    if log[i]["epoch"] != log[i - 1]["epoch"]]
        out[tag] = res_dict(r) | {
            "restart_checks": restarts,
            "log": [[e["iteration"], e["epoch"], e["rel_primal"], e["rel_dual"], e["rel_box"],
                     e["rel_gap"], e["sigma"]] for e in log],
            "solve_time_s": r.solve_time,
        }
        print("C1", tag, r.status.value, r.iterations, r.restarts, r.objective, r.solve_time)
    with open(os.path.join(HERE, "c1_trajectory.json"), "w") as fh:
        json.dump(out, fh)


def make_c2():
    """C2 + 500 triples: PTDF flow rows of up to ~1,900 entries, so the
    engine's padded index-free rows and A^T y flow panels are on the path
    (C1's ~225-entry flow rows are below both thresholds)."""
    doc, mon, lpa = scuc.build_config("C2", n_triples=500)
    lp = ref_lp(lpa.indptr, lpa.indices, lpa.data, lpa.shape, lpa.rhs, lpa.cost,
                lpa.lower, lpa.upper, lpa.n_eq)
    out = {"digest": lpa.digest(), "shape": list(lpa.shape), "nnz": lpa.nnz}
    r = solve_record(lp, tolerance=1e-4, ruiz=False, precision=lp_kernel.Precision.FP64,
                     log_residuals=True)
    log = r.residual_log
    out["fp64"] = res_dict(r) | {
        "log": [[e["iteration"], e["epoch"], e["rel_primal"], e["rel_dual"], e["rel_box"],
                 e["rel_gap"], e["sigma"]] for e in log],
        "solve_time_s": r.solve_time,
    }
    print("C2", r.status.value, r.iterations, r.restarts, r.objective, r.solve_time)
    with open(os.path.join(HERE, "c2_trajectory.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    if not a.only or a.only == "kat":
        make_kat()
    if not a.only or a.only == "random":
        make_random()
    if not a.only or a.only == "scuc":
        make_scuc_small()
    if a.c1 or a.only == "c1":
        make_c1()
    if a.only == "c2":
        make_c2()
