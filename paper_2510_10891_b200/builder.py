"""Drop-in model construction for the reference driver.

``build_model`` replaces ``scuckit.formulation.build_model``
(``formulation.py:215-413``) and ``compute_ptdf`` replaces
``scuckit.instance.compute_ptdf`` (``instance.py:241-267``).  ``hprlp.install``
rebinds both wherever the reference imported them by name (the driver calls
them at ``driver.py:210`` and ``:249-250``), so a filtering pass builds its
MILP in seconds instead of minutes (597 s -> a few s at C4) and the PTDF
tables come from one factorisation instead of one per contingency.

``build_model`` returns the reference's own ``MilpModel`` / ``VariableMap`` /
``StandardFormLp`` / ``SparseMatrix`` objects: the rows, bounds, costs,
row tags and column tags are the reference's exactly (tests/test_builder.py
compares them field by field); the arithmetic is the vectorised restatement
in ``scuc.build_relaxation``.  ``compute_ptdf`` returns the reference's
``PtdfTable``: base rows from one dense solve of the reduced susceptance
matrix, contingency tables by the LODF update (``scuc._lodf_rows``); the
values agree with the reference's per-contingency refactorisation to
rounding (1e-12), not bit for bit -- LAPACK itself is not reproducible
across thread counts, so neither is the reference's table.
"""

from __future__ import annotations

import numpy as np

from . import scuc
from .lp import lazy_csc_matrix


class _TableRows:
    """``scuc.PtdfRows``' read interface over a ``PtdfTable`` (the driver hands
    ``build_model`` a table object; ``formulation.py:354`` reads rows of it)."""

    def __init__(self, table):
        self.table = table

    def row(self, lpos: int, key: str) -> np.ndarray:
        return self.table.table(key)[lpos]


def _row_tags(instance, n_rows_flow_triples) -> list:
    """Row tags in build_model's row order (formulation.py:243-369)."""
    gids = [g.gid for g in instance.generators]
    T = int(instance.n_periods)
    ts = range(T)
    tags = []
    for fmt in ("logic-eq", "seg-sum", "cost-def"):
        tags += [f"{fmt} g={g} t={t}" for g in gids for t in ts]
    tags += [f"balance t={t}" for t in ts]
    for fmt in ("logic-ineq", "min-up", "min-down", "prod-limit", "ramp-up", "ramp-down"):
        tags += [f"{fmt} g={g} t={t}" for g in gids for t in ts]
    for gen in instance.generators:
        tags += [f"seg-cap g={gen.gid} t={t} h={h}" for t in ts for h in range(gen.n_segments)]
    for lid, t, key in n_rows_flow_triples:
        tags.append(f"flow-lo l={lid} t={t} c={key}")
        tags.append(f"flow-hi l={lid} t={t} c={key}")
    return tags


def _col_tags(instance, vmap) -> list:
    """Column tags of build_model (formulation.py:378-403), in column order."""
    gids = [g.gid for g in instance.generators]
    T = int(instance.n_periods)
    ts = range(T)
    tags = []
    for label in ("u", "v", "w", "pprime"):
        tags += [f"{label} g={g} t={t}" for g in gids for t in ts]
    for gen in instance.generators:
        tags += [f"seg g={gen.gid} t={t} h={h}" for t in ts for h in range(gen.n_segments)]
    tags += [f"cost g={g} t={t}" for g in gids for t in ts]
    tags += [f"dpen b={b.bid} t={t}" for b in instance.buses for t in ts]
    if len(tags) != vmap.n_cols:
        raise AssertionError("column tag count does not match the variable map")
    return tags


def build_model(instance, monitored=(), ptdf=None):
    """``formulation.build_model`` (formulation.py:215-413): the SCUC MILP over
    the monitored flow triples, as the reference's (MilpModel, VariableMap)."""
    import scipy.sparse as sp
    from scuckit import formulation as F
    from scuckit import lp_kernel as K
    vmap = F.VariableMap(instance)
    n_t = instance.n_periods
    monitored = sorted(set(monitored))
    if monitored:
        valid_keys = set(instance.contingency_keys())
        line_pos = instance.network.line_index()
        for lid, t, key in monitored:                            # :229-233
            if lid not in line_pos or not (0 <= t < n_t) or key not in valid_keys:
                raise F.ModelError(f"monitored triple ({lid}, {t}, {key}) is out of range")
        if ptdf is None:
            ptdf = instance.ptdf or compute_ptdf(instance.network)
    arrays = scuc.Instance.from_scuckit(instance)
    lpa = scuc.build_relaxation(arrays, monitored,
                                ptdf=_TableRows(ptdf) if monitored else None)
    csr = sp.csr_matrix((lpa.data, lpa.indices, lpa.indptr), shape=lpa.shape)
    lp = K.StandardFormLp(matrix=lazy_csc_matrix(K.SparseMatrix, csr), rhs=lpa.rhs, cost=lpa.cost,
                          lower=lpa.lower, upper=lpa.upper, n_eq=lpa.n_eq,
                          row_tags=_row_tags(instance, monitored),
                          col_tags=_col_tags(instance, vmap))
    return F.MilpModel(lp, vmap.binary_mask.copy(), vmap), vmap


def _connected(n_b, fb, tb, skip=None) -> bool:
    """instance._connected (instance.py:176-196): BFS from bus 0."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    keep = np.ones(len(fb), bool)
    if skip is not None:
        keep[skip] = False
    g = sp.coo_matrix((np.ones(int(keep.sum())), (fb[keep], tb[keep])), shape=(n_b, n_b))
    return connected_components(g, directed=False)[0] == 1


def compute_ptdf(network, device=None):
    """``instance.compute_ptdf`` (instance.py:241-267): PTDF tables for the
    base topology and every single-line contingency, as the reference's
    ``PtdfTable``, with the same connectivity and |PTDF| <= 1 checks and
    errors.  One base solve (on the current CUDA device when there is one);
    contingency tables by the LODF update."""
    from scuckit import instance as I
    bidx = network.bus_index()
    lidx = network.line_index()
    n_b = len(network.buses)
    fb = np.array([bidx[ln.from_bus] for ln in network.lines], dtype=np.int64)
    tb = np.array([bidx[ln.to_bus] for ln in network.lines], dtype=np.int64)
    react = np.array([ln.reactance for ln in network.lines], dtype=np.float64)
    ref = bidx[network.reference_bus]
    if not _connected(n_b, fb, tb):
        raise I.InstanceError("network", "base topology is disconnected")
    if device is None:
        try:
            import torch
            device = "cuda" if torch.cuda.is_available() else None
        except ImportError:
            device = None
    lines = list(range(len(fb)))
    base = scuc._ptdf_rows_direct(n_b, fb, tb, react, ref, lines, device=device)
    tables = {I.BASE_CASE: base}
    for cont in network.contingencies:
        k = lidx[cont.line]
        if not _connected(n_b, fb, tb, skip=k):
            raise I.InstanceError(cont.cid, f"contingency isolates bus (outage of line {cont.line})")
        tables[cont.cid] = scuc._lodf_rows(base, base[k], lines, k, fb, tb, ref)
    for key, mat in tables.items():
        if np.max(np.abs(mat), initial=0.0) > 1.0 + I._PTDF_SANITY_EPS:
            raise I.InstanceError(f"ptdf[{key}]", "PTDF magnitude exceeds 1; check reactances")
    return I.PtdfTable(tables, [ln.lid for ln in network.lines],
                       [b.bid for b in network.buses], network.reference_bus)
