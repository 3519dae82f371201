"""Row-partitioned HPR on CPU ranks — TEST INFRASTRUCTURE ONLY.

This restates the reference HPR solve (``scuckit/hprlp.py:332-455``, using
the same building blocks as ``oracle/hpr_oracle.py``) in the row-partitioned
form that the multi-GPU engine runs. Each rank owns one
row block from ``paper_2510_10891_b200.partition`` and one slice of the
columns (chunk = ceil(n / world_size), rank r owns [r·chunk, (r+1)·chunk)).
The collectives are ``torch.distributed``: gloo in the CPU tests, NCCL in
the engine. Every collective of the device implementation appears here, in
the same place:

* scaling: column ∞-norms (MAX), column 1-norms (SUM), ‖rhs‖² (SUM);
* power method: Aᵀv partials (SUM) and ‖A Aᵀ v‖² (SUM);
* iteration: the Aᵀy partials are reduce-scattered to the column owners,
  each rank updates its own x / z slice, and x̃ is all-gathered for the
  local A x̃ product and dual update;
* check: the master bar x is all-gathered, the row-side KKT sums (SUM) and
  the Aᵀ y_m partials (reduce-scatter) are taken, the column-side sums of
  each slice are all-reduced, and the controller runs replicated on the
  reduced sums, so every rank takes the same restart / σ / stopping
  decisions.

``tests/test_partitioned.py`` runs it with world_size 2 over gloo and
compares it with the single-process oracle.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch
import torch.distributed as dist

from oracle import hpr_oracle as O


def _allreduce(a: np.ndarray, op=dist.ReduceOp.SUM) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t, op=op)
    return t.numpy()


def _allsum(v: float) -> float:
    return float(_allreduce(np.array([v]))[0])


def _slice(n: int):
    ws, r = dist.get_world_size(), dist.get_rank()
    chunk = -(-n // ws)
    c0 = min(n, r * chunk)
    return chunk, c0, min(n, c0 + chunk)


def _reduce_scatter(a: np.ndarray) -> np.ndarray:
    """Sum of the ranks' n-vectors, this rank's owned chunk only."""
    ws = dist.get_world_size()
    chunk, c0, c1 = _slice(a.shape[0])
    full = np.zeros(chunk * ws)
    full[:a.shape[0]] = a
    out = torch.zeros(chunk, dtype=torch.float64)
    dist.reduce_scatter(out, list(torch.from_numpy(full).split(chunk)))
    return out.numpy()[:c1 - c0]


def _all_gather(part: np.ndarray, n: int) -> np.ndarray:
    """The n-vector whose owned chunks are `part` on their ranks."""
    ws = dist.get_world_size()
    chunk, c0, c1 = _slice(n)
    buf = np.zeros(chunk)
    buf[:c1 - c0] = part
    outs = [torch.zeros(chunk, dtype=torch.float64) for _ in range(ws)]
    dist.all_gather(outs, torch.from_numpy(buf))
    return torch.cat(outs).numpy()[:n]


class Block:
    """Rank-local rows (equalities first) with replicated column data."""

    def __init__(self, a_rows, rhs, cost, lower, upper, n_eq, offset):
        self.a = O.Csr(a_rows)
        self.rhs, self.cost = np.asarray(rhs, float), np.asarray(cost, float)
        self.lower, self.upper = np.asarray(lower, float), np.asarray(upper, float)
        self.n_eq, self.offset = int(n_eq), float(offset)


def _scaling(b: Block, cfg):
    a = b.a.cast(np.float64)
    m, n = a.shape
    rs, cs = np.ones(m), np.ones(n)
    if cfg.ruiz:
        for _ in range(cfg.ruiz_iters):
            r = a.abs_row_max()
            c = _allreduce(a.abs_col_max(), dist.ReduceOp.MAX)
            r = 1.0 / np.sqrt(np.where(r > 0, r, 1.0))
            c = 1.0 / np.sqrt(np.where(c > 0, c, 1.0))
            rs *= r
            cs *= c
            a = a.times_diag(r, c)
            dev = max(np.abs(1.0 - r).max(initial=0.0), np.abs(1.0 - c).max(initial=0.0))
            if _allreduce(np.array([dev]), dist.ReduceOp.MAX)[0] < 1e-6:
                break
    if cfg.pock_chambolle:
        r = a.abs_row_sum()
        c = _allreduce(a.abs_col_sum())
        r = 1.0 / np.sqrt(np.where(r > 0, r, 1.0))
        c = 1.0 / np.sqrt(np.where(c > 0, c, 1.0))
        rs *= r
        cs *= c
        a = a.times_diag(r, c)
    rhs = b.rhs * rs
    cost = b.cost * cs
    lo = np.where(np.isfinite(b.lower), b.lower / cs, b.lower)
    up = np.where(np.isfinite(b.upper), b.upper / cs, b.upper)
    if cfg.normalize_rhs_objective:
        fin = rhs[np.isfinite(rhs)]
        bsc = 1.0 + float(np.sqrt(_allsum(float(fin @ fin))))
        csc = 1.0 + float(np.linalg.norm(cost))
    else:
        bsc = csc = 1.0
    work = Block(a.a, rhs / bsc, cost / csc, np.where(np.isfinite(lo), lo / bsc, lo),
                 np.where(np.isfinite(up), up / bsc, up), b.n_eq, 0.0)
    return work, rs, cs, bsc, csc


def _power(a: O.Csr, v0_local, tol, max_iter, inflation):
    v = v0_local / np.sqrt(_allsum(float(v0_local @ v0_local)))
    lam, prev = 0.0, -1.0
    for _ in range(max_iter):
        u = _allreduce(a.aty(v))
        w = a.ax(u)
        lam = float(np.sqrt(_allsum(float(w @ w))))
        v = w / lam
        if abs(lam - prev) <= tol * max(lam, 1e-300):
            break
        prev = lam
    return lam * (1.0 + tol if inflation is None else inflation)


def solve(block: Block, global_rows: np.ndarray, m_total: int, cfg) -> dict:
    """Partitioned HPR solve on this rank; returns the best master triple
    (x, z replicated; y for the local rows) and the trajectory summary."""
    cfg = O.OracleConfig.from_any(cfg)
    w, rs, cs, bsc, csc = _scaling(block, cfg)
    rng = np.random.default_rng(cfg.seed)
    v0 = rng.standard_normal(m_total)[global_rows]
    lam = _power(w.a, v0, cfg.power_tol, cfg.power_max_iter, cfg.power_inflation)
    rn = np.sqrt(_allsum(float(w.rhs @ w.rhs)))
    cn = float(np.linalg.norm(w.cost))
    sigma = cfg.sigma0 if cfg.sigma0 is not None else (rn / cn if rn > 1e-12 and cn > 1e-12 else 1.0)
    denom = 1.0 + np.sqrt(_allsum(float(block.rhs @ block.rhs))) + float(np.linalg.norm(block.cost))
    m, n = w.a.shape
    x = O.box(np.zeros(n), w.lower, w.upper)
    y, z = np.zeros(m), np.zeros(n)
    ax_, ay_, az_ = x.copy(), y.copy(), z.copy()
    norm_a = float(np.sqrt(lam))

    chunk, c0, c1 = _slice(n)
    sl = slice(c0, c1)

    def kkt(bx_s, by, bz_s):
        """KKT of the bar triple; bx_s / bz_s are this rank's column slices."""
        xm_s, ym, zm_s = bx_s * cs[sl] * bsc, by * rs * csc, bz_s * csc / cs[sl]
        xm = _all_gather(xm_s, n)                                   # for the local A x_m
        pv = ym - O.dual_cone(ym - block.a.ax(xm) + block.rhs, block.n_eq)
        aty_s = _reduce_scatter(block.a.aty(ym))
        rows = _allreduce(np.array([pv @ pv, block.rhs @ ym]))
        dv = block.cost[sl] - aty_s - zm_s
        bv = xm_s - O.box(xm_s - zm_s, block.lower[sl], block.upper[sl])
        zp, zn = np.maximum(zm_s, 0.0), np.minimum(zm_s, 0.0)
        lo_t = np.where(np.isfinite(block.lower[sl]), block.lower[sl] * zp, 0.0)
        up_t = np.where(np.isfinite(block.upper[sl]), block.upper[sl] * zn, 0.0)
        cols = _allreduce(np.array([dv @ dv, bv @ bv, float(block.cost[sl] @ xm_s),
                                    float(lo_t.sum() + up_t.sum())]))
        pobj = cols[2] + block.offset
        dobj = rows[1] + cols[3] + block.offset
        rp, rb, rd = np.sqrt(rows[0]) / denom, np.sqrt(cols[1]) / denom, np.sqrt(cols[0]) / denom
        gap = abs(pobj - dobj)
        rg = gap / (1.0 + abs(pobj) + abs(dobj))
        return max(rp, rb, rd, rg), pobj, (xm, ym, _all_gather(zm_s, n))

    x_s, z_s = x[sl].copy(), z[sl].copy()
    ax_s, az_s = x_s.copy(), z_s.copy()
    best, pobj, tri = kkt(x_s, y, z_s)
    last_restart = epoch_min = best
    best_tri, best_obj = tri, pobj
    k = total = last_imp = restarts = 0
    status = "iteration-limit"
    if best <= cfg.tolerance:
        return dict(status="optimal-tolerance", iterations=0, restarts=0, objective=pobj,
                    lam=lam, x=tri[0], y=tri[1], z=tri[2], sigma=sigma)
    while total < cfg.max_iterations:
        p_s = _reduce_scatter(w.a.aty(y))                         # Aᵀy partials -> owners
        g = x_s + sigma * (p_s - w.cost[sl])
        bx_s = O.box(g, w.lower[sl], w.upper[sl])
        bz_s = (bx_s - g) / sigma
        xt_s = 2.0 * bx_s - x_s
        xt = _all_gather(xt_s, n)                                   # x~ for the local rows
        by = O.dual_cone(y + (1.0 / (lam * sigma)) * (w.rhs - w.a.ax(xt)), w.n_eq)
        t = 1.0 / (k + 2.0)
        x_s = t * ax_s + (1.0 - t) * xt_s
        y = t * ay_ + (1.0 - t) * (2.0 * by - y)
        z_s = t * az_s + (1.0 - t) * (2.0 * bz_s - z_s)
        k += 1
        total += 1
        if total % cfg.check_every:
            continue
        res, pobj, tri = kkt(bx_s, by, bz_s)
        if res < best:
            best, best_tri, best_obj = res, tri, pobj
        if res < epoch_min * (1.0 - 1e-12):
            epoch_min, last_imp = res, total
        if res <= cfg.tolerance:
            best_tri, best_obj = tri, pobj
            status = "optimal-tolerance"
            break
        if res <= cfg.restart_beta * last_restart or total - last_imp >= cfg.restart_stall:
            dx = np.sqrt(_allsum(float((bx_s - ax_s) @ (bx_s - ax_s))))
            dy = np.sqrt(_allsum(float((by - ay_) @ (by - ay_))))
            if dx > 1e-14 and dy > 1e-14 and norm_a > 0:
                sigma *= float(np.clip((dx / (norm_a * dy * sigma)) ** cfg.sigma_damping, 0.25, 4.0))
            ax_s, ay_, az_s = bx_s.copy(), by.copy(), bz_s.copy()
            x_s, y, z_s = bx_s.copy(), by.copy(), bz_s.copy()
            k = 0
            restarts += 1
            last_restart = epoch_min = res
            last_imp = total
    return dict(status=status, iterations=total, restarts=restarts, objective=best_obj, lam=lam,
                x=best_tri[0], y=best_tri[1], z=best_tri[2], sigma=sigma)


def block_from_lp(lp, blk):
    csr = lp.matrix.csr if hasattr(lp, "matrix") else lp.csr()
    return Block(sp.csr_matrix(csr[blk.rows]), np.asarray(lp.rhs)[blk.rows], lp.cost, lp.lower,
                 lp.upper, blk.n_eq, float(getattr(lp, "offset", 0.0)))
