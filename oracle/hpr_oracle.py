"""CPU oracle for the HPR-LP hot path — TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy/scipy restatement of the reference's
HPR solver (``scuckit/hprlp.py``) and its sparse substrate
(``scuckit/lp_kernel.py``).  It exists to *check* the CUDA engine, and to
time the reference algorithm on the GPU box's host cores where the reference
package itself is not installed.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may
import it; the product path (``paper_2510_10891_b200``) never does.

Parity pinning: ``tests/test_oracle_golden.py`` checks this restatement
against golden vectors produced by running the unmodified reference in the
build container (``tests/golden/make_golden.py``): bit-identical results on
the SPEC known-answer tests and small random LPs, identical iteration /
restart trajectories on SCUC relaxations.

Arithmetic follows the reference operation by operation (same scipy CSR
products, same numpy elementwise order, FP32 work arrays with 64-bit
norms), so an FP64 oracle run reproduces the reference's iterates exactly.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

OPTIMAL = "optimal-tolerance"
ITERATION_LIMIT = "iteration-limit"
TIME_LIMIT = "time-limit"
NUMERICAL_FAILURE = "numerical-failure"


@dataclass
class OracleConfig:
    """Field-for-field ``SolverConfig`` (``hprlp.py:34-60``); precision is
    "fp64" or "fp32"."""

    tolerance: float = 1e-6
    max_iterations: int = 400_000
    time_limit: float | None = None
    precision: str = "fp64"
    sigma0: float | None = None
    restart_beta: float = 0.2
    restart_stall: int = 500
    sigma_damping: float = 0.5
    ruiz: bool = True
    ruiz_iters: int = 10
    pock_chambolle: bool = True
    normalize_rhs_objective: bool = True
    check_every: int = 16
    power_tol: float = 1e-4
    power_inflation: float = 1.01
    power_max_iter: int = 5000
    seed: int = 0
    log_residuals: bool = False
    log_every_iteration: bool = False

    @classmethod
    def from_any(cls, cfg) -> "OracleConfig":
        if cfg is None:
            return cls()
        if isinstance(cfg, cls):
            return cfg
        if isinstance(cfg, dict):
            return cls(**cfg)
        kw = {k: getattr(cfg, k) for k in cls.__dataclass_fields__ if hasattr(cfg, k)}
        p = kw.get("precision")
        if p is not None and not isinstance(p, str):
            kw["precision"] = p.value
        return cls(**kw)

    @property
    def dtype(self):
        return np.float32 if self.precision == "fp32" else np.float64


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def norm64(a) -> float:                              # lp_kernel.py:39-41
    return float(np.linalg.norm(_f64(a)))


def dot64(a, b) -> float:                            # lp_kernel.py:34-36
    return float(np.dot(_f64(a), _f64(b)))


class Csr:
    """A canonical CSR matrix with its transpose kept as a CSR of A^T built
    from the CSC layout (``lp_kernel.py:52-62``); products are scipy's."""

    def __init__(self, a, dtype=np.float64):
        a = sp.csr_matrix(a, dtype=dtype)
        a.sum_duplicates()
        a.eliminate_zeros()
        a.sort_indices()
        self.a = a
        csc = a.tocsc()
        csc.sort_indices()
        self.csc = csc
        self.at = csc.T
        self.shape = a.shape

    def ax(self, x):                                  # lp_kernel.py:78-82
        if x.shape[0] != self.shape[1]:
            raise ValueError("matvec dimension mismatch")
        return self.a @ x

    def aty(self, y):                                 # lp_kernel.py:84-88
        if y.shape[0] != self.shape[0]:
            raise ValueError("matvec_t dimension mismatch")
        return self.at @ y

    def cast(self, dtype):
        return self if self.a.dtype == dtype else Csr(self.a, dtype)

    def abs_row_max(self):                            # lp_kernel.py:105-110 (ord=inf)
        return abs(self.a.astype(np.float64)).max(axis=1).toarray().ravel()

    def abs_col_max(self):
        return abs(self.csc.astype(np.float64)).max(axis=0).toarray().ravel()

    def abs_row_sum(self):                            # ord=1
        return np.asarray(abs(self.a.astype(np.float64)).sum(axis=1)).ravel()

    def abs_col_sum(self):
        return np.asarray(abs(self.csc.astype(np.float64)).sum(axis=0)).ravel()

    def times_diag(self, r, c):
        """diag(r) A diag(c) with the reference's rounding: (a*r_i)*c_j
        (``lp_kernel.py:118-122``)."""
        a = self.a.astype(np.float64).tocoo()
        data = (a.data * np.asarray(r, np.float64)[a.row]) * np.asarray(c, np.float64)[a.col]
        return Csr(sp.csr_matrix((data, (a.row, a.col)), shape=a.shape), self.a.dtype)


def power_lambda(a: Csr, tol, max_iter, seed, inflation) -> float:
    """lambda_max(A A^T) by the implicit power method (``lp_kernel.py:138-175``)."""
    if a.a.nnz == 0:
        raise ValueError("power_method requires a nonzero matrix")
    a64 = a.cast(np.float64)
    m = a64.shape[0]
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(m)
    v /= norm64(v)
    lam, prev, ok = 0.0, -1.0, False
    for _ in range(max_iter):
        wv = a64.ax(a64.aty(v))
        lam = norm64(wv)
        if lam <= 0.0:
            v = rng.standard_normal(m)
            v /= norm64(v)
            prev = -1.0
            continue
        v = wv / lam
        if abs(lam - prev) <= tol * max(lam, 1e-300):
            ok = True
            break
        prev = lam
    if not ok:
        warnings.warn("power method did not converge", RuntimeWarning)
    return lam * (1.0 + tol if inflation is None else inflation)


def box(x, lo, up):                                   # lp_kernel.py:128-130
    return np.minimum(np.maximum(x, lo), up)


def dual_cone(y, n_eq):                               # lp_kernel.py:208-213
    out = np.array(y, copy=True)
    out[n_eq:] = np.maximum(out[n_eq:], 0.0)
    return out


@dataclass
class Problem:
    a: Csr
    rhs: np.ndarray
    cost: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    n_eq: int
    offset: float = 0.0

    @classmethod
    def from_lp(cls, lp) -> "Problem":
        """From a reference ``StandardFormLp`` or any duck-typed equivalent
        (``.matrix.csr``), or from ``paper_2510_10891_b200.scuc.LpArrays``."""
        mat = lp.csr() if hasattr(lp, "indptr") else lp.matrix.csr
        return cls(Csr(mat), _f64(lp.rhs), _f64(lp.cost), _f64(lp.lower), _f64(lp.upper),
                   int(lp.n_eq), float(getattr(lp, "offset", 0.0)))


@dataclass
class Kkt:
    """``KktResidual`` (``hprlp.py:63-95``)."""

    primal: float
    box: float
    dual: float
    rel_primal: float
    rel_box: float
    rel_dual: float
    primal_objective: float
    dual_objective: float
    gap: float
    rel_gap: float

    @property
    def max_rel(self):
        return max(self.rel_primal, self.rel_box, self.rel_dual, self.rel_gap)

    @property
    def combined(self):
        return float(np.sqrt(self.primal ** 2 + self.box ** 2 + self.dual ** 2))


def kkt(p: Problem, x, y, z) -> Kkt:
    """KKT residual on master (unscaled FP64) data (``hprlp.py:98-139``)."""
    x, y, z = _f64(x), _f64(y), _f64(z)
    pv = y - dual_cone(y - p.a.ax(x) + p.rhs, p.n_eq)
    bv = x - box(x - z, p.lower, p.upper)
    dv = p.cost - p.a.aty(y) - z
    den = 1.0 + norm64(p.rhs) + norm64(p.cost)
    r_p, r_b, r_d = norm64(pv), norm64(bv), norm64(dv)
    pobj = dot64(p.cost, x) + p.offset
    zp, zm = np.maximum(z, 0.0), np.minimum(z, 0.0)
    lo_t = np.where(np.isfinite(p.lower), p.lower * zp, 0.0)
    up_t = np.where(np.isfinite(p.upper), p.upper * zm, 0.0)
    dobj = dot64(p.rhs, y) + float(lo_t.sum() + up_t.sum()) + p.offset
    gap = abs(pobj - dobj)
    return Kkt(r_p, r_b, r_d, r_p / den, r_b / den, r_d / den, pobj, dobj, gap,
               gap / (1.0 + abs(pobj) + abs(dobj)))


class Scaling:
    """Ruiz -> Pock-Chambolle -> rhs/objective normalisation
    (``hprlp.py:210-276``)."""

    def __init__(self, p: Problem, cfg: OracleConfig):
        a = p.a.cast(np.float64)
        m, n = a.shape
        rs, cs = np.ones(m), np.ones(n)
        if cfg.ruiz:
            for _ in range(cfg.ruiz_iters):
                r, c = a.abs_row_max(), a.abs_col_max()
                r = 1.0 / np.sqrt(np.where(r > 0, r, 1.0))
                c = 1.0 / np.sqrt(np.where(c > 0, c, 1.0))
                rs *= r
                cs *= c
                a = a.times_diag(r, c)
                if max(np.abs(1.0 - r).max(initial=0.0), np.abs(1.0 - c).max(initial=0.0)) < 1e-6:
                    break
        if cfg.pock_chambolle:
            r, c = a.abs_row_sum(), a.abs_col_sum()
            r = 1.0 / np.sqrt(np.where(r > 0, r, 1.0))
            c = 1.0 / np.sqrt(np.where(c > 0, c, 1.0))
            rs *= r
            cs *= c
            a = a.times_diag(r, c)
        rhs = p.rhs * rs
        cost = p.cost * cs
        lo = np.where(np.isfinite(p.lower), p.lower / cs, p.lower)
        up = np.where(np.isfinite(p.upper), p.upper / cs, p.upper)
        if cfg.normalize_rhs_objective:
            self.b_scale = 1.0 + float(np.linalg.norm(rhs[np.isfinite(rhs)]))
            self.c_scale = 1.0 + float(np.linalg.norm(cost))
        else:
            self.b_scale = self.c_scale = 1.0
        self.rs, self.cs = rs, cs
        self.work = Problem(a, rhs / self.b_scale, cost / self.c_scale,
                            np.where(np.isfinite(lo), lo / self.b_scale, lo),
                            np.where(np.isfinite(up), up / self.b_scale, up), p.n_eq)

    def to_work(self, x, y, z):
        return (x / (self.cs * self.b_scale), y / (self.rs * self.c_scale),
                z * self.cs / self.c_scale)

    def to_master(self, x, y, z):
        return (_f64(x) * self.cs * self.b_scale, _f64(y) * self.rs * self.c_scale,
                _f64(z) * self.c_scale / self.cs)


@dataclass
class OracleResult:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    status: str
    objective: float
    kkt: Kkt
    iterations: int
    restarts: int
    solve_time: float
    sigma_final: float
    lam: float
    residual_log: list = field(default_factory=list)
    rate_log: list = field(default_factory=list)
    precision_used: str = "fp64"
    fp64_fallback: bool = False
    restart_log: list = field(default_factory=list)   # (iteration, kind, sigma_after)

    @property
    def converged(self):
        return self.status == OPTIMAL


class HprIterate:
    """Work-space iteration state and one HPR step (``hprlp.py:142-207``)."""

    def __init__(self, x, y, z, sigma, lam, dtype):
        self.x = np.array(x, dtype=dtype)
        self.y = np.array(y, dtype=dtype)
        self.z = np.array(z, dtype=dtype)
        self.ax_, self.ay_, self.az_ = self.x.copy(), self.y.copy(), self.z.copy()
        self.bx = self.by = self.bz = None
        self.sigma, self.lam, self.k, self.total, self.epoch = sigma, lam, 0, 0, 0

    def step(self, w: Problem):
        s = self.sigma
        g = self.x + s * (w.a.aty(self.y) - w.cost)
        bx = box(g, w.lower, w.upper)
        bz = (bx - g) / s
        xt = 2.0 * bx - self.x
        by = dual_cone(self.y + (1.0 / (self.lam * s)) * (w.rhs - w.a.ax(xt)), w.n_eq)
        t = 1.0 / (self.k + 2.0)
        yh = 2.0 * by - self.y
        zh = 2.0 * bz - self.z
        self.x = t * self.ax_ + (1.0 - t) * xt
        self.y = t * self.ay_ + (1.0 - t) * yh
        self.z = t * self.az_ + (1.0 - t) * zh
        self.bx, self.by, self.bz = bx, by, bz
        self.k += 1
        self.total += 1

    def restart(self):
        self.ax_, self.ay_, self.az_ = self.bx.copy(), self.by.copy(), self.bz.copy()
        self.x, self.y, self.z = self.bx.copy(), self.by.copy(), self.bz.copy()
        self.k = 0
        self.epoch += 1


def solve(lp, config=None, start=None) -> OracleResult:
    """``hprlp.solve`` (``hprlp.py:319-329``): one attempt, FP64 retry after
    an FP32 numerical failure."""
    cfg = OracleConfig.from_any(config)
    p = lp if isinstance(lp, Problem) else Problem.from_lp(lp)
    res = _solve_once(p, cfg, start)
    if res.status == NUMERICAL_FAILURE and cfg.precision == "fp32":
        cfg64 = OracleConfig(**{**cfg.__dict__, "precision": "fp64"})
        res = _solve_once(p, cfg64, start)
        res.fp64_fallback = True
    return res


def setup(p: Problem, cfg: OracleConfig):
    """Scaling, work-precision copy, lambda, sigma0 (``hprlp.py:335-355``)."""
    sc = Scaling(p, cfg)
    dt = cfg.dtype
    w = sc.work
    if dt == np.float32:
        w = Problem(w.a.cast(np.float32), w.rhs.astype(dt), w.cost.astype(dt),
                    w.lower.astype(dt), w.upper.astype(dt), w.n_eq)
    lam = power_lambda(sc.work.a, cfg.power_tol, cfg.power_max_iter, cfg.seed,
                       cfg.power_inflation)
    rn, cn = norm64(sc.work.rhs), norm64(sc.work.cost)
    if cfg.sigma0 is not None:
        sigma = cfg.sigma0
    elif rn > 1e-12 and cn > 1e-12:
        sigma = rn / cn
    else:
        sigma = 1.0
    return sc, w, lam, sigma


def _solve_once(p: Problem, cfg: OracleConfig, start) -> OracleResult:
    t0 = time.perf_counter()
    sc, w, lam, sigma = setup(p, cfg)
    m, n = p.a.shape
    if start is None:
        x0, y0, z0 = np.zeros(n), np.zeros(m), np.zeros(n)
    else:
        x0, y0, z0 = sc.to_work(*[_f64(v) for v in start])
    x0 = box(x0, sc.work.lower, sc.work.upper)
    st = HprIterate(x0, y0, z0, sigma, lam, cfg.dtype)

    def master(xw, yw, zw):
        tri = sc.to_master(xw, yw, zw)
        return kkt(p, *tri), tri

    r0, tri0 = master(st.x, st.y, st.z)
    best, best_tri = r0, tri0
    last_restart, epoch_min, last_imp = r0.max_rel, r0.max_rel, 0
    norm_a = float(np.sqrt(lam))
    rlog, rate, rstlog = [], [], []
    restarts = 0
    status = ITERATION_LIMIT
    every = 1 if cfg.log_every_iteration else max(1, cfg.check_every)

    def result(tri, res, its):
        return OracleResult(tri[0], tri[1], tri[2], status, dot64(p.cost, tri[0]) + p.offset,
                            res, its, restarts, time.perf_counter() - t0, st.sigma, lam,
                            rlog, rate, cfg.precision, False, rstlog)

    if r0.max_rel <= cfg.tolerance:
        status = OPTIMAL
        return result(tri0, r0, 0)

    while True:
        if st.total >= cfg.max_iterations:
            status = ITERATION_LIMIT
            break
        if cfg.time_limit is not None and time.perf_counter() - t0 > cfg.time_limit:
            status = TIME_LIMIT
            break
        st.step(w)
        if st.total % every:
            continue
        if not (np.isfinite(st.bx).all() and np.isfinite(st.by).all() and np.isfinite(st.bz).all()):
            status = NUMERICAL_FAILURE
            break
        res, tri = master(st.bx, st.by, st.bz)
        if cfg.log_every_iteration:
            rate.append((st.epoch, st.k, res.combined))
        if cfg.log_residuals or cfg.log_every_iteration:
            rlog.append({"iteration": st.total, "epoch": st.epoch,
                         "rel_primal": res.rel_primal, "rel_dual": res.rel_dual,
                         "rel_box": res.rel_box, "rel_gap": res.rel_gap, "sigma": st.sigma})
        if res.max_rel < best.max_rel:
            best, best_tri = res, tri
        if res.max_rel < epoch_min * (1.0 - 1e-12):
            epoch_min, last_imp = res.max_rel, st.total
        if res.max_rel <= cfg.tolerance:
            best, best_tri = res, tri
            status = OPTIMAL
            break
        suff = res.max_rel <= cfg.restart_beta * last_restart
        stall = st.total - last_imp >= cfg.restart_stall
        if suff or stall:
            dx = norm64(st.bx - st.ax_)
            dy = norm64(st.by - st.ay_)
            if dx > 1e-14 and dy > 1e-14 and norm_a > 0:
                ratio = dx / (norm_a * dy * st.sigma)
                st.sigma *= float(np.clip(ratio ** cfg.sigma_damping, 0.25, 4.0))
            st.restart()
            restarts += 1
            rstlog.append((st.total, "sufficient" if suff else "stall", st.sigma))
            last_restart = epoch_min = res.max_rel
            last_imp = st.total
    return result(best_tri, best, st.total)
