"""Row partitioning of the HPR LP across GPUs.

A is split by rows into ``world_size`` blocks; every rank keeps all n columns,
so x, z and the column data are replicated and only the Aᵀy partials need a
collective. Three rules shape the blocks:

* **Locality.** Rows are ordered by period first, using the engine's
  period-major key: the smallest "long-row key" of their columns. Each block
  then holds whole periods' structural rows together with the PTDF flow rows
  of those periods (`formulation.py:351-369`). This matches the split
  "by time period and line-flow block" that the north star names.
* **Balance.** Contiguous cuts equalise nonzeros, not rows.
* **Twins stay together.** A (lo, hi) flow-row pair is never split, so each
  rank can still fold it (hpr_update.cuh).

Each block is re-emitted as a standard-form LP with its equality rows first:
``n_eq_d`` counts the block's equalities. ``StandardFormLp`` semantics
(`lp_kernel.py:178-213`) are preserved block by block.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class RowBlock:
    rank: int
    rows: np.ndarray          # original row indices, equalities first
    n_eq: int                 # equalities among them
    nnz: int


def _twin_next(indptr, indices, data, i) -> bool:
    """Row i+1 is the exact negation of row i (same pattern)."""
    a0, a1 = indptr[i], indptr[i + 1]
    b0, b1 = indptr[i + 1], indptr[i + 2]
    if a1 - a0 != b1 - b0 or a1 == a0:
        return False
    return bool(np.array_equal(indices[a0:a1], indices[b0:b1])
                and np.array_equal(data[b0:b1], -data[a0:a1]))


def period_key(indptr, indices, n, long_row=256):
    """Column key = first long row touching the column (the balance row of
    its period for SCUC); row key = smallest key of its columns.  Mirrors
    hpr_engine.cu: compute_order."""
    m = len(indptr) - 1
    lens = np.diff(indptr)
    inf = np.iinfo(np.int64).max
    ckey = np.full(n, inf, dtype=np.int64)
    for i in np.flatnonzero(lens > long_row):
        cols = indices[indptr[i]:indptr[i + 1]]
        sel = ckey[cols] == inf
        ckey[cols[sel]] = i
    corder = np.argsort(ckey, kind="stable")
    crank = np.empty(n, dtype=np.int64)
    crank[corder] = np.arange(n)
    rkey = np.full(m, inf, dtype=np.int64)
    rows = np.repeat(np.arange(m), lens)
    np.minimum.at(rkey, rows, crank[indices])
    return rkey


def partition_rows(indptr, indices, data, n_eq: int, n: int, world_size: int) -> list:
    """Balanced, period-grouped, twin-preserving row blocks."""
    indptr = np.asarray(indptr)
    m = len(indptr) - 1
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    rkey = period_key(indptr, indices, n)
    # ordering units: single rows or twin pairs (inequality block only)
    units = []
    i = 0
    while i < m:
        if i >= n_eq and i + 1 < m and _twin_next(indptr, indices, data, i):
            units.append((i, 2))
            i += 2
        else:
            units.append((i, 1))
            i += 1
    ukey = np.array([rkey[u[0]] for u in units])
    order = np.argsort(ukey, kind="stable")
    lens = np.diff(indptr)
    unnz = np.array([lens[u[0]:u[0] + u[1]].sum() for u in units])
    cum = np.cumsum(unnz[order])
    total = int(cum[-1]) if len(cum) else 0
    blocks = []
    start = 0
    for r in range(world_size):
        target = total * (r + 1) / world_size
        stop = int(np.searchsorted(cum, target, side="right")) if r < world_size - 1 else len(order)
        stop = max(stop, start)
        sel = order[start:stop]
        rows = np.concatenate([np.arange(units[u][0], units[u][0] + units[u][1]) for u in sel]) \
            if len(sel) else np.zeros(0, dtype=np.int64)
        rows = np.sort(rows)                      # original order inside a block
        eq = rows[rows < n_eq]
        ineq = rows[rows >= n_eq]
        rows = np.concatenate([eq, ineq]).astype(np.int64)
        blocks.append(RowBlock(rank=r, rows=rows, n_eq=int(eq.size), nnz=int(lens[rows].sum())))
        start = stop
    covered = np.sort(np.concatenate([b.rows for b in blocks]))
    if not np.array_equal(covered, np.arange(m)):
        raise AssertionError("row partition does not cover every row exactly once")
    return blocks


def block_lp(lp, block: RowBlock):
    """The rank-local LP: rows of the block (equalities first), all columns."""
    from .lp import SparseMatrix, StandardFormLp
    csr = lp.matrix.csr if hasattr(lp, "matrix") else lp.csr()
    sub = csr[block.rows]
    return StandardFormLp(matrix=SparseMatrix(sub), rhs=np.asarray(lp.rhs)[block.rows],
                          cost=np.asarray(lp.cost), lower=np.asarray(lp.lower),
                          upper=np.asarray(lp.upper), n_eq=block.n_eq,
                          offset=float(getattr(lp, "offset", 0.0)))
