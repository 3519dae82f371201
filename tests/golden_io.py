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
