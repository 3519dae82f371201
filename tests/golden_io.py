"""Loaders for the committed golden fixtures (tests/golden/)."""

import json
import os

import numpy as np
import scipy.sparse as sp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def kat():
    with open(os.path.join(GOLDEN, "kat.json")) as fh:
        return json.load(fh)


class FixtureLp:
    """Minimal StandardFormLp-shaped object (``.matrix.csr``)."""

    def __init__(self, indptr, indices, data, shape, rhs, cost, lower, upper, n_eq, offset=0.0):
        from paper_2510_10891_b200.lp import SparseMatrix
        self.matrix = SparseMatrix(sp.csr_matrix((data, indices, indptr), shape=tuple(shape)))
        self.rhs = np.asarray(rhs, float)
        self.cost = np.asarray(cost, float)
        self.lower = np.asarray(lower, float)
        self.upper = np.asarray(upper, float)
        self.n_eq = int(n_eq)
        self.offset = float(offset)

    @property
    def n_rows(self):
        return self.matrix.shape[0]

    @property
    def n_cols(self):
        return self.matrix.shape[1]

    def objective(self, x):
        return float(np.dot(self.cost, x)) + self.offset


def random_lps():
    z = np.load(os.path.join(GOLDEN, "random_lps.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    out = []
    for i, rec in enumerate(meta):
        lp = FixtureLp(*(z[f"lp{i}_{k}"] for k in ("indptr", "indices", "data", "shape", "rhs",
                                                   "cost", "lower", "upper")),
                       int(z[f"lp{i}_n_eq"]))
        res = {}
        for tag in ("fp64", "fp32", "fp64_noruiz_log"):
            r = dict(rec[tag])
            r["x"], r["y"], r["z"] = (z[f"lp{i}_{tag}_{c}"] for c in "xyz")
            if f"lp{i}_{tag}_log" in z:
                r["log"] = z[f"lp{i}_{tag}_log"]
            res[tag] = r
        out.append((lp, rec, res))
    return out


def scuc_small():
    z = np.load(os.path.join(GOLDEN, "scuc_small.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    lp = FixtureLp(z["indptr"], z["indices"], z["data"], z["shape"], z["rhs"], z["cost"],
                   z["lower"], z["upper"], int(z["n_eq"]))
    res = {}
    for tag in ("fp64_1e4", "fp64_1e6_ruiz", "fp32_1e4"):
        r = dict(meta[tag])
        r["x"], r["y"], r["z"] = (z[f"{tag}_{c}"] for c in "xyz")
        r["log"] = z[f"{tag}_log"]
        res[tag] = r
    return lp, meta, res


def c1():
    p = os.path.join(GOLDEN, "c1_trajectory.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        return json.load(fh)


def c2():
    p = os.path.join(GOLDEN, "c2_trajectory.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        return json.load(fh)


def warm_starts():
    """[(start (x, y, z), {"fp64": rec, "fp32": rec})] for random_lps()[:6]
    (tests/golden/make_warm_golden.py)."""
    z = np.load(os.path.join(GOLDEN, "warm_starts.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    return [(tuple(z[f"lp{i}_{c}0"] for c in "xyz"), rec) for i, rec in enumerate(meta)]


LOG_COLS = ("iteration", "epoch", "rel_primal", "rel_dual", "rel_box", "rel_gap", "sigma")


def log_rows(result) -> np.ndarray:
    """A SolveResult's residual log as the golden files store it: one row
    [iteration, epoch, rel_primal, rel_dual, rel_box, rel_gap, sigma] per check."""
    return np.array([[e[k] for k in LOG_COLS] for e in result.residual_log], dtype=np.float64)


def restart_list(rows, beta=0.2, stall=500):
    """Restarts read off a residual log (hprlp.py:422-446): the epoch advances
    at the check that restarted.  The kind is "beta" when max_rel <= beta x
    (max_rel at the last restart), else "stall" (no improvement of the epoch
    minimum for `stall` iterations).  The log does not carry the initial
    residual, so in epoch 0 a restart that also meets the stall rule is
    labelled "stall".  [(check iteration, kind, sigma at the check, sigma
    after)], the shape of make_c4_golden.restart_list."""
    rows = np.asarray(rows, dtype=np.float64)
    out = []
    last = None                    # max_rel at the last restart
    emin, last_imp = np.inf, 0
    for i in range(len(rows)):
        it, mr = int(rows[i, 0]), float(rows[i, 2:6].max())
        if mr < emin * (1.0 - 1e-12):
            emin, last_imp = mr, it
        if i + 1 < len(rows) and rows[i + 1, 1] != rows[i, 1]:
            if last is not None:
                kind = "beta" if mr <= beta * last else "stall"
            else:
                kind = "stall" if it - last_imp >= stall else "beta"
            out.append((it, kind, float(rows[i, 6]), float(rows[i + 1, 6])))
            last, emin, last_imp = mr, mr, it
    return out


def trajectory_diff(mine, ref) -> dict:
    """Check-by-check comparison of two logs (rows as in log_rows): the first
    check where iteration or epoch differ, and the worst relative difference
    of the residual and sigma columns over the common prefix."""
    mine, ref = np.asarray(mine, float), np.asarray(ref, float)
    n = min(len(mine), len(ref))
    same = np.all(mine[:n, :2] == ref[:n, :2], axis=1)
    first_bad = int(np.argmin(same)) if not same.all() else n
    a, b = mine[:first_bad, 2:], ref[:first_bad, 2:]
    rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
    rel[(a == b)] = 0.0
    # row-relative: each residual's difference over the row's max_rel (the
    # quantity the tolerance and restart tests read), so a component that is
    # ~0 (rel_box is often 1e-17) does not dominate
    scale = np.maximum(b[:, :4].max(axis=1, initial=0.0), 1e-300)
    rowrel = np.abs(a[:, :4] - b[:, :4]).max(axis=1, initial=0.0) / scale
    rowrel = np.maximum(rowrel, rel[:, 4]) if len(rel) else rowrel
    return {"rows_mine": len(mine), "rows_ref": len(ref), "aligned_rows": first_bad,
            "max_rel_resid": float(rel[:, :4].max(initial=0.0)),
            "max_rel_sigma": float(rel[:, 4].max(initial=0.0)),
            "max_row_rel": float(rowrel.max(initial=0.0)),
            "max_rel_by_row": rowrel.tolist()}


def c4_window():
    p = os.path.join(GOLDEN, "c4_window.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        return json.load(fh)
