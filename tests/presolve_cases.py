"""Seeded presolve cases shared by tests/test_presolve.py and
tests/golden/make_presolve_golden.py: small MILPs that exercise every rule of
the reference presolve (presolve.py:94-209) — tightening in both directions,
integral rounding, redundant / empty rows, infinite bounds — and each of its
infeasibility certificates."""

import hashlib

import numpy as np


def random_case(seed, classes):
    """(model, kind) built with the given classes: a namespace with
    SparseMatrix, StandardFormLp and MilpModel (reference or mirror)."""
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(6, 40)), int(rng.integers(5, 30))
    a = rng.standard_normal((m, n)) * (rng.uniform(size=(m, n)) < 0.3)
    a[rng.uniform(size=(m, n)) < 0.1] = rng.choice([-1.0, 1.0, 2.0])
    kind = seed % 5
    if kind == 1:
        a[m // 2] = 0.0                                   # empty row
    lower = np.where(rng.uniform(size=n) < 0.15, -np.inf, -rng.uniform(0, 2, n))
    upper = np.where(rng.uniform(size=n) < 0.15, np.inf, rng.uniform(0, 2, n))
    integ = rng.uniform(size=n) < 0.4
    lower[integ] = np.maximum(lower[integ], 0.0)
    upper[integ] = 1.0
    x = np.clip(rng.uniform(-1, 1, n), np.where(np.isfinite(lower), lower, -1),
                np.where(np.isfinite(upper), upper, 1))
    x[integ] = np.round(np.clip(x[integ], 0, 1))
    rhs = a @ x
    n_eq = int(rng.integers(0, m // 3 + 1))
    rhs[n_eq:] -= rng.uniform(0, 0.5, m - n_eq) * (rng.uniform(size=m - n_eq) < 0.7)
    if kind == 2:
        rhs[n_eq:] += 50.0 * (rng.uniform(size=m - n_eq) < 0.05)     # row infeasibility
    if kind == 3 and n_eq:
        rhs[0] = -1e3                                                 # eq min-activity
    if kind == 1:
        rhs[m // 2] = 0.0 if seed % 2 else (1.0 if m // 2 >= n_eq else 0.0)
    if kind == 4 and integ.any():
        j0 = int(np.flatnonzero(integ)[0])                            # integral rounding
        extra = np.zeros((1, n))                                      # empties a domain:
        extra[0, j0] = 1.0                                            # x_j0 = 0.5 (equality)
        a = np.vstack([extra, a])
        rhs = np.concatenate([[0.5], rhs])
        m += 1
        n_eq += 1
    cost = rng.standard_normal(n)
    lp = classes.StandardFormLp(matrix=classes.SparseMatrix(a), rhs=rhs, cost=cost,
                                lower=lower, upper=upper, n_eq=n_eq, offset=0.25,
                                row_tags=[f"r{i}" for i in range(m)] if seed % 3 else [],
                                col_tags=[f"c{j}" for j in range(n)] if seed % 3 else [])
    return classes.MilpModel(lp, integ, None), kind


def digest(result):
    """Digest of (reduced model or LP, ReductionLog): every field the
    reference produces, bit for bit."""
    red, log = result
    lp = red.lp if hasattr(red, "lp") else red
    h = hashlib.sha256()
    c = lp.matrix.csr

    def put(a):
        h.update(np.ascontiguousarray(a).tobytes())

    for arr in (c.indptr.astype(np.int64), c.indices.astype(np.int64), c.data, lp.rhs, lp.cost,
                lp.lower, lp.upper, np.asarray(log.kept_cols, np.int64),
                np.asarray(log.kept_rows, np.int64)):
        put(arr)
    if hasattr(red, "integrality"):
        put(np.asarray(red.integrality, dtype=np.uint8))
    h.update(repr((lp.n_eq, lp.offset, list(lp.row_tags), list(lp.col_tags),
                   sorted(log.fixed_values.items()), log.removed_rows, log.bound_changes,
                   log.objective_delta, log.infeasible)).encode())
    return h.hexdigest()
