"""Drop-in HPR-LP solver backed by the sm_100a engine (libhprlp_b200.so).

Mirrors the reference module ``scuckit.hprlp`` (``pkg/src/scuckit/hprlp.py``)
name for name — ``SolverConfig``, ``KktResidual``, ``SolveStatus``,
``SolveResult``, ``HprState``, ``hpr_iterate``, ``kkt_residual``,
``solve``, ``write_iteration_log`` — with the same argument meaning and
error behaviour.  All arithmetic runs on the GPU through the C-ABI
(``include/hprlp_b200.h``); this module only marshals arrays.

``install()`` rebinds ``scuckit.hprlp.solve`` to :func:`solve`.
``scuckit.lp_backends.solve_lp`` looks ``hprlp.solve`` up at call time
(``lp_backends.py:36``), so the transmission-filtering driver, successive
fixing (``fixing.py:164``) and the B&B node LPs (``milp_bb.py:241``) all
route to the GPU with no edit to the reference.  Results are then built from
the reference's own dataclasses, so ``res.converged`` / ``res.status.value``
behave exactly as before.
"""

from __future__ import annotations

import enum
import logging
import time
import weakref
from dataclasses import dataclass, field, replace

import numpy as np

from . import _capi
from .lp import Precision

log = logging.getLogger(__name__)


class SolveStatus(enum.Enum):
    """``hprlp.SolveStatus`` (hprlp.py:27-31)."""

    OPTIMAL = "optimal-tolerance"
    ITERATION_LIMIT = "iteration-limit"
    TIME_LIMIT = "time-limit"
    NUMERICAL_FAILURE = "numerical-failure"


_STATUS_BY_CODE = {_capi.HPR_OPTIMAL: "OPTIMAL", _capi.HPR_ITERATION_LIMIT: "ITERATION_LIMIT",
                   _capi.HPR_TIME_LIMIT: "TIME_LIMIT",
                   _capi.HPR_NUMERICAL_FAILURE: "NUMERICAL_FAILURE"}


@dataclass
class SolverConfig:
    """``hprlp.SolverConfig`` (hprlp.py:34-60), same fields and validation."""

    tolerance: float = 1e-6
    max_iterations: int = 400_000
    time_limit: float | None = None
    precision: Precision = Precision.FP64
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

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if not 0.0 < self.restart_beta < 1.0:
            raise ValueError("restart_beta must lie in (0, 1)")


@dataclass
class KktResidual:
    """``hprlp.KktResidual`` (hprlp.py:63-95)."""

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
    def combined(self) -> float:
        return float(np.sqrt(self.primal ** 2 + self.box ** 2 + self.dual ** 2))

    @property
    def max_rel(self) -> float:
        return max(self.rel_primal, self.rel_box, self.rel_dual, self.rel_gap)

    def converged(self, tolerance: float) -> bool:
        return self.max_rel <= tolerance


@dataclass
class SolveResult:
    """``hprlp.SolveResult`` (hprlp.py:279-300)."""

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    status: SolveStatus
    objective: float
    kkt: KktResidual
    iterations: int
    restarts: int
    solve_time: float
    sigma_final: float
    lam: float
    residual_log: list = field(default_factory=list)
    rate_log: list = field(default_factory=list)
    precision_used: Precision = Precision.FP64
    fp64_fallback: bool = False
    # engine telemetry (not in the reference record)
    device_stats: dict = field(default_factory=dict)

    @property
    def converged(self) -> bool:
        return self.status.value == "optimal-tolerance"


@dataclass
class HprState:
    """``hprlp.HprState`` (hprlp.py:142-181)."""

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    anchor_x: np.ndarray
    anchor_y: np.ndarray
    anchor_z: np.ndarray
    bar_x: np.ndarray | None = None
    bar_y: np.ndarray | None = None
    bar_z: np.ndarray | None = None
    sigma: float = 1.0
    lam: float = 1.0
    k: int = 0
    total_iterations: int = 0
    epoch: int = 0
    last_restart_residual: float | None = None

    @classmethod
    def from_point(cls, x, y, z, sigma=1.0, lam=1.0, dtype=np.float64) -> "HprState":
        x = np.array(x, dtype=dtype)
        y = np.array(y, dtype=dtype)
        z = np.array(z, dtype=dtype)
        return cls(x=x, y=y, z=z, anchor_x=x.copy(), anchor_y=y.copy(), anchor_z=z.copy(),
                   sigma=sigma, lam=lam)

    def restart(self) -> None:
        self.anchor_x, self.anchor_y, self.anchor_z = (self.bar_x.copy(), self.bar_y.copy(),
                                                       self.bar_z.copy())
        self.x, self.y, self.z = self.bar_x.copy(), self.bar_y.copy(), self.bar_z.copy()
        self.k = 0
        self.epoch += 1


# ---------------------------------------------------------------------------
# result classes: ours, or the reference's after install()
# ---------------------------------------------------------------------------

class _Classes:
    status = SolveStatus
    result = SolveResult
    kkt = KktResidual
    precision = Precision


_CLS = _Classes()


def _precision_value(p) -> str:
    return p.value if hasattr(p, "value") else str(p)


def _precision_member(value: str):
    return _CLS.precision(value)


# ---------------------------------------------------------------------------
# engine: one LP uploaded to one GPU
# ---------------------------------------------------------------------------

def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class Engine:
    """An LP resident on one B200: CSR of A and A^T, tile plans, workspace.

    The device workspace is a torch uint8 tensor (PyTorch owns the memory);
    the engine's kernels run on a private CUDA stream of the handle."""

    def __init__(self, lp, device: int | None = None, reorder: bool = True, fold: bool = True,
                 runs: bool = True, panels: bool = True, comm=None, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("the HPR engine needs a CUDA device (no CPU fallback)")
        t_create = time.perf_counter()
        self._lib = _capi.load()
        csr = lp.matrix.csr
        m, n = csr.shape
        self.m, self.n = int(m), int(n)
        self.n_eq = int(lp.n_eq)
        self.offset = float(getattr(lp, "offset", 0.0))
        self._keep = [_i32(csr.indptr), _i32(csr.indices), _f64(csr.data)]
        tparts = [None, None, None]          # A^T is built on the device (hpr_layout.cuh)
        vecs = [_f64(lp.rhs), _f64(lp.cost), _f64(lp.lower), _f64(lp.upper)]
        if vecs[0].shape != (m,) or any(v.shape != (n,) for v in vecs[1:]):
            raise ValueError("LP vector lengths do not match the matrix shape")
        self._keep += vecs
        P = _capi.ptr
        self._prob = _capi.Problem(self.m, self.n, self.n_eq, int(csr.nnz),
                                   P(self._keep[0]), P(self._keep[1]), P(self._keep[2]),
                                   P(tparts[0]), P(tparts[1]), P(tparts[2]),
                                   P(vecs[0]), P(vecs[1]), P(vecs[2]), P(vecs[3]), self.offset)
        nbytes = _capi.C.c_size_t(0)
        _capi.check(self._lib.hpr_workspace_bytes(_capi.C.byref(self._prob), _capi.C.byref(nbytes)))
        dev = torch.cuda.current_device() if device is None else int(device)
        self.device = dev
        self._ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=f"cuda:{dev}")
        flags = ((0 if reorder else _capi.HPR_FLAG_NO_REORDER)
                 | (0 if fold else _capi.HPR_FLAG_NO_FOLD)
                 | (0 if runs else _capi.HPR_FLAG_NO_RUNS)
                 | (0 if panels else _capi.HPR_FLAG_NO_PANELS))
        ncomm, world, rank = (None, 1, 0) if comm is None else (comm.handle, comm.world_size,
                                                                 comm.rank)
        # stream: a torch.cuda.Stream to run on (e.g. a low-priority one); None =
        # a private stream at the device's greatest priority
        self._stream = stream
        sp = None if stream is None else _capi.C.c_void_p(stream.cuda_stream)
        opt = _capi.Options(dev, sp, _capi.C.c_void_p(self._ws.data_ptr()), int(nbytes.value),
                            flags, ncomm, world, rank)
        h = _capi.C.c_void_p()
        _capi.check(self._lib.hpr_create(_capi.C.byref(self._prob), _capi.C.byref(opt),
                                         _capi.C.byref(h)))
        self._h = h
        self.nnz = int(csr.nnz)
        self.workspace_bytes = int(nbytes.value)
        self.create_seconds = time.perf_counter() - t_create   # host arrays -> resident layout
        self._create_reported = False

    def close(self):
        if getattr(self, "_h", None):
            self._lib.hpr_destroy(self._h)
            self._h = None
            self._ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- kernels exposed for the reference's substrate API -----------------
    def matvec(self, x, transpose=False):
        x = _f64(x)
        if x.shape[0] != (self.m if transpose else self.n):
            raise ValueError(f"matvec dimension mismatch: A is {(self.m, self.n)}, "
                             f"vector has {x.shape[0]}")
        out = np.empty(self.n if transpose else self.m)
        _capi.check(self._lib.hpr_matvec(self._h, int(transpose), _capi.ptr(x), _capi.ptr(out)))
        return out

    def kkt(self, x, y, z) -> _capi.Kkt:
        x, y, z = _f64(x), _f64(y), _f64(z)
        k = _capi.Kkt()
        _capi.check(self._lib.hpr_kkt_residual(self._h, _capi.ptr(x), _capi.ptr(y),
                                               _capi.ptr(z), _capi.C.byref(k)))
        return k

    def power(self, tol, max_iter, seed, inflation):
        rng = np.random.default_rng(seed)
        starts = [rng.standard_normal(self.m)]
        while True:
            buf = _f64(np.concatenate(starts))
            lam = _capi.C.c_double()
            it, cv = _capi.C.c_int32(), _capi.C.c_int32()
            code = self._lib.hpr_power_method(
                self._h, float(tol), int(max_iter), -1.0 if inflation is None else float(inflation),
                _capi.ptr(buf), len(starts), _capi.C.byref(lam), _capi.C.byref(it),
                _capi.C.byref(cv))
            if code == _capi.HPR_ERR_POWER_NULL:
                starts.append(rng.standard_normal(self.m))
                continue
            _capi.check(code)
            return lam.value, it.value, bool(cv.value)

    def iterate(self, precision, sigma, lam, k, x, y, z, ax, ay, az):
        args = [_f64(v) for v in (x, y, z, ax, ay, az)]
        outs = [np.empty(self.n), np.empty(self.m), np.empty(self.n),
                np.empty(self.n), np.empty(self.m), np.empty(self.n)]
        _capi.check(self._lib.hpr_iterate(self._h, precision, float(sigma), float(lam), int(k),
                                          *[_capi.ptr(a) for a in args],
                                          *[_capi.ptr(o) for o in outs]))
        return outs

    def resume(self, more_iterations, tolerance=0.0) -> _capi.Stats:
        """Continue the last solve's device state (benchmark support)."""
        st = _capi.Stats()
        _capi.check(self._lib.hpr_resume(self._h, int(more_iterations), float(tolerance),
                                         _capi.C.byref(st)))
        return st

    def layout(self) -> dict:
        """Device layout: folded rows / nonzeros, tile counts, workspace bytes."""
        lay = _capi.Layout()
        _capi.check(self._lib.hpr_get_layout(self._h, _capi.C.byref(lay)))
        return {k: getattr(lay, k) for k, _ in lay._fields_}

    def bench_kernel(self, which: int, reps: int = 20, in_iteration: bool = False) -> float:
        """Average device seconds of one iteration kernel (hpr_bench_kernel:
        0: A x~ product, 1: A^T y product, 2: primal update, 3: dual update,
        4: one KKT check block, 5 / 6: the fused pair).  `in_iteration`: each
        timed launch is followed by the iteration's other kernels, so the
        caches hold what they hold in the loop."""
        sec = _capi.C.c_double()
        w = int(which) | (_capi.HPR_BENCH_IN_ITERATION if in_iteration else 0)
        _capi.check(self._lib.hpr_bench_kernel(self._h, w, int(reps), _capi.C.byref(sec)))
        return sec.value

    def solve_raw(self, config, start=None, time_elapsed=0.0, rows=None, m_total=None):
        """One ``_solve_once`` on the device; returns (x, y, z, Stats, log).
        For a row block of a partitioned solve, `rows` / `m_total` select the
        block's slice of the global power-method start vector."""
        cfg = config
        prec = _precision_value(cfg.precision)
        rng = np.random.default_rng(cfg.seed)

        def draw():
            v = rng.standard_normal(self.m if rows is None else m_total)
            return v if rows is None else v[rows]

        starts = [draw()]
        x = np.empty(self.n)
        y = np.empty(self.m)
        z = np.empty(self.n)
        x0 = y0 = z0 = None
        if start is not None:
            # numpy broadcasting as in _ScaleMaps.to_work (hprlp.py:266-270): a
            # scalar spreads, a wrong length raises ValueError
            x0, y0, z0 = (_f64(np.broadcast_to(np.asarray(v, dtype=np.float64), (k,)))
                          for v, k in zip(start, (self.n, self.m, self.n)))
        while True:
            pbuf = _f64(np.concatenate(starts))
            prm = _capi.Params(
                tolerance=float(cfg.tolerance), max_iterations=int(cfg.max_iterations),
                time_limit=-1.0 if cfg.time_limit is None else float(cfg.time_limit),
                time_elapsed=float(time_elapsed),
                precision=_capi.HPR_FP32 if prec == "fp32" else _capi.HPR_FP64,
                has_sigma0=int(cfg.sigma0 is not None),
                sigma0=0.0 if cfg.sigma0 is None else float(cfg.sigma0),
                restart_beta=float(cfg.restart_beta), restart_stall=int(cfg.restart_stall),
                sigma_damping=float(cfg.sigma_damping), ruiz=int(bool(cfg.ruiz)),
                ruiz_iters=int(cfg.ruiz_iters), pock_chambolle=int(bool(cfg.pock_chambolle)),
                normalize_rhs_objective=int(bool(cfg.normalize_rhs_objective)),
                check_every=int(cfg.check_every), power_tol=float(cfg.power_tol),
                power_inflation=-1.0 if cfg.power_inflation is None else float(cfg.power_inflation),
                power_max_iter=int(cfg.power_max_iter), power_start=_capi.ptr(pbuf),
                power_start_count=len(starts), log_residuals=int(bool(cfg.log_residuals)),
                log_every_iteration=int(bool(cfg.log_every_iteration)))
            st = _capi.Stats()
            code = self._lib.hpr_solve(self._h, _capi.C.byref(prm), _capi.ptr(x0), _capi.ptr(y0),
                                       _capi.ptr(z0), _capi.ptr(x), _capi.ptr(y), _capi.ptr(z),
                                       _capi.C.byref(st))
            if code == _capi.HPR_ERR_POWER_NULL:
                starts.append(draw())
                continue
            if code == _capi.HPR_ERR_EMPTY:
                raise ValueError("power_method requires a nonzero matrix")
            if code == _capi.HPR_ERR_INVALID:
                raise ValueError(self._lib.hpr_last_error().decode())
            _capi.check(code)
            break
        recs = []
        if st.n_log:
            buf = (_capi.LogRecord * st.n_log)()
            nout = _capi.C.c_int64()
            _capi.check(self._lib.hpr_get_log(self._h, buf, st.n_log, _capi.C.byref(nout)))
            recs = list(buf)
        return x, y, z, st, recs


_ENGINES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def engine_for(lp) -> Engine:
    """Engine for an LP, cached per (immutable) matrix object and vector set."""
    key = lp.matrix
    sig = (id(lp.rhs), id(lp.cost), id(lp.lower), id(lp.upper), int(lp.n_eq),
           float(getattr(lp, "offset", 0.0)))
    try:
        ent = _ENGINES.get(key)
    except TypeError:
        ent = None
    if ent is not None and ent[0] == sig and all(
            np.array_equal(a, b) for a, b in zip(ent[2], (lp.rhs, lp.cost, lp.lower, lp.upper))):
        return ent[1]
    eng = Engine(lp)
    try:
        _ENGINES[key] = (sig, eng, tuple(np.array(v, copy=True) for v in
                                         (lp.rhs, lp.cost, lp.lower, lp.upper)))
    except TypeError:
        pass
    return eng


# ---------------------------------------------------------------------------
# the reference API
# ---------------------------------------------------------------------------

def _kkt_obj(k: _capi.Kkt):
    return _CLS.kkt(primal=k.primal, box=k.box, dual=k.dual, rel_primal=k.rel_primal,
                    rel_box=k.rel_box, rel_dual=k.rel_dual,
                    primal_objective=k.primal_objective, dual_objective=k.dual_objective,
                    gap=k.gap, rel_gap=k.rel_gap)


def kkt_residual(x, y, z, lp):
    """``hprlp.kkt_residual`` (hprlp.py:116-139) evaluated on the GPU."""
    return _kkt_obj(engine_for(lp).kkt(x, y, z))


def hpr_iterate(state, lp):
    """``hprlp.hpr_iterate`` (hprlp.py:184-207): one step on the GPU in the
    state's dtype.  Mutates and returns `state`."""
    prec = _capi.HPR_FP32 if np.asarray(state.x).dtype == np.float32 else _capi.HPR_FP64
    dt = np.float32 if prec == _capi.HPR_FP32 else np.float64
    x, y, z, bx, by, bz = engine_for(lp).iterate(prec, state.sigma, state.lam, state.k, state.x,
                                                 state.y, state.z, state.anchor_x,
                                                 state.anchor_y, state.anchor_z)
    state.x, state.y, state.z = x.astype(dt), y.astype(dt), z.astype(dt)
    state.bar_x, state.bar_y, state.bar_z = bx.astype(dt), by.astype(dt), bz.astype(dt)
    state.k += 1
    state.total_iterations += 1
    return state


def power_method(lp_or_matrix, tol=1e-4, max_iter=1000, seed=0, inflation=None) -> float:
    """``lp_kernel.power_method`` (lp_kernel.py:138-175) on the GPU."""
    from .lp import StandardFormLp
    lp = lp_or_matrix
    if not hasattr(lp, "matrix"):
        m, n = lp.shape
        lp = StandardFormLp(matrix=lp, rhs=np.zeros(m), cost=np.zeros(n), lower=np.zeros(n),
                            upper=np.zeros(n))
    if lp.matrix.csr.nnz == 0:
        raise ValueError("power_method requires a nonzero matrix")
    lam, _, conv = engine_for(lp).power(tol, max_iter, seed, inflation)
    if not conv:
        import warnings
        warnings.warn("power method reached max_iter without converging; "
                      "returning the inflated last estimate", RuntimeWarning)
    return lam


def _assemble(lp, config, x, y, z, st, recs, t_start, stats):
    """A SolveResult (hprlp.py:448-455) from one device solve: best triple,
    status, KKT of the returned point, and both logs (hprlp.py:412-420)."""
    status = getattr(_CLS.status, _STATUS_BY_CODE[st.status])
    residual_log, rate_log = [], []
    if config.log_every_iteration:
        rate_log = [(r.epoch, r.k, float(np.sqrt(r.primal ** 2 + r.box ** 2 + r.dual ** 2)))
                    for r in recs]
    if config.log_residuals or config.log_every_iteration:
        residual_log = [{"iteration": r.iteration, "epoch": r.epoch, "rel_primal": r.rel_primal,
                         "rel_dual": r.rel_dual, "rel_box": r.rel_box, "rel_gap": r.rel_gap,
                         "sigma": r.sigma} for r in recs]
    objective = float(np.dot(_f64(lp.cost), x)) + float(getattr(lp, "offset", 0.0))
    res = _CLS.result(x=x, y=y, z=z, status=status, objective=objective, kkt=_kkt_obj(st.kkt),
                      iterations=int(st.iterations), restarts=int(st.restarts),
                      solve_time=time.perf_counter() - t_start, sigma_final=st.sigma_final,
                      lam=st.lam, residual_log=residual_log, rate_log=rate_log,
                      precision_used=_precision_member(_precision_value(config.precision)))
    try:
        res.device_stats = stats
    except AttributeError:
        pass
    return res


def _solve_once(lp, config, start, t_start, engine=None):
    eng = engine_for(lp) if engine is None else engine
    x, y, z, st, recs = eng.solve_raw(config, start, time.perf_counter() - t_start)
    stats = {"setup_seconds": st.setup_seconds, "loop_seconds": st.loop_seconds,
             # the engine build this call paid for (0 when the cached engine was reused)
             "create_seconds": 0.0 if eng._create_reported else eng.create_seconds,
             "gpu_launches": int(st.gpu_launches), "power_iterations": st.power_iterations,
             "checks": int(st.checks), "device_objective": st.objective}
    eng._create_reported = True
    return _assemble(lp, config, x, y, z, st, recs, t_start, stats)


def _with_fp64_retry(config, run):
    """``solve``'s FP32 -> FP64 retry (hprlp.py:324-328): `run(cfg, t_start)`
    is one solve; an FP32 numerical failure reruns it in FP64."""
    result = run(config, time.perf_counter())
    if (result.status.value == "numerical-failure"
            and _precision_value(config.precision) == "fp32"):
        log.warning("FP32 solve failed numerically; retrying in FP64")
        cfg64 = replace(config, precision=type(config.precision)("fp64")) \
            if hasattr(config, "__dataclass_fields__") else config
        result = run(cfg64, time.perf_counter())
        result.fp64_fallback = True
    return result


def solve(lp, config=None, start=None):
    """``hprlp.solve`` (hprlp.py:319-329) on the GPU: one device solve, and an
    FP64 retry when an FP32 solve loses finiteness."""
    return _with_fp64_retry(config or SolverConfig(),
                            lambda cfg, t0: _solve_once(lp, cfg, start, t0))


def solve_many(lps, config=None, starts=None, workers: int | None = None) -> list:
    """Several independent LP solves on one GPU at once (SURVEY §8(f) rank 4:
    the node LPs of a branch-and-bound frontier, ``milp_bb.py:204-253``, or
    any set of fixing-round LPs).  Each LP gets its own engine, so its own
    CUDA stream and graph (``hprlp_b200.h``: distinct handles are
    independent); one host thread per solve drives it, and ctypes releases
    the GIL inside the C-ABI, so the solves overlap on the device.  Each
    result is exactly what :func:`solve` returns for that LP alone (same
    kernels, same per-LP order of operations); only the wall clock is shared.
    Small LPs (C1/C2 size) run in the engine's launch-latency regime, which
    is where overlapping several of them pays."""
    from concurrent.futures import ThreadPoolExecutor
    lps = list(lps)
    if starts is None:
        starts = [None] * len(lps)
    if len(starts) != len(lps):
        raise ValueError("starts must match lps")
    if not lps:
        return []
    import torch
    config = config or SolverConfig()
    dev = torch.cuda.current_device()
    workers = max(1, min(workers or 8, len(lps)))

    def one(a):
        # a private engine per entry: two entries never share a handle (a
        # handle is not thread-safe), and the caller's device, not the
        # worker thread's default 0, holds it
        torch.cuda.set_device(dev)
        eng = Engine(a[0], device=dev)
        try:
            return _with_fp64_retry(config,
                                    lambda cfg, t0: _solve_once(a[0], cfg, a[1], t0, engine=eng))
        finally:
            eng.close()

    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(one, zip(lps, starts)))


def write_iteration_log(path, result, solve_id: str = "solve") -> None:
    """``hprlp.write_iteration_log`` (hprlp.py:303-316)."""
    import csv
    import os
    new = not os.path.exists(path)
    with open(path, "a", newline="") as fh:
        w = csv.writer(fh)
        if new:
            w.writerow(["solve_id", "iteration", "epoch", "rel_primal", "rel_dual", "rel_box",
                        "rel_gap", "sigma"])
        for rec in result.residual_log:
            w.writerow([solve_id, rec["iteration"], rec["epoch"], rec["rel_primal"],
                        rec["rel_dual"], rec["rel_box"], rec["rel_gap"], rec["sigma"]])


# ---------------------------------------------------------------------------
# row-partitioned solve across the GPUs of one node
# ---------------------------------------------------------------------------

class NcclComm:
    """An NCCL communicator for the engine, bootstrapped over an initialised
    torch.distributed process group (rank 0's unique id is broadcast)."""

    def __init__(self, group=None, device: int | None = None):
        import torch
        import torch.distributed as dist
        self.world_size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        lib = _capi.load()
        uid = (_capi.C.c_uint8 * 128)()
        if self.rank == 0:
            _capi.check(lib.hpr_nccl_unique_id(_capi.C.byref(uid)))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        uid = (_capi.C.c_uint8 * 128).from_buffer_copy(box[0])
        dev = torch.cuda.current_device() if device is None else int(device)
        h = _capi.C.c_void_p()
        _capi.check(lib.hpr_nccl_comm_init(_capi.C.byref(uid), self.world_size, self.rank, dev,
                                           _capi.C.byref(h)))
        self.handle = h
        self._lib = lib

    def close(self):
        if self.handle:
            self._lib.hpr_nccl_comm_destroy(self.handle)
            self.handle = None


def solve_partitioned(lp, config=None, start=None, comm: NcclComm | None = None, group=None):
    """``solve`` with A row-partitioned over the ranks of `group` (one GPU per
    rank).  Every rank passes the same full LP; each keeps its row block
    (paper_2510_10891_b200.partition).  x, z come back replicated and y is
    gathered, so every rank returns the full SolveResult -- with the same
    logs and the same FP32 -> FP64 retry as :func:`solve` (the retry decision
    is taken on replicated controller state, so all ranks take it together)."""
    import torch.distributed as dist
    from . import partition
    own = comm is None
    comm = comm or NcclComm(group)
    try:
        csr = lp.matrix.csr
        blocks = partition.partition_rows(csr.indptr, csr.indices, csr.data, int(lp.n_eq),
                                          csr.shape[1], comm.world_size)
        blk = blocks[comm.rank]
        blp = partition.block_lp(lp, blk)
        eng = Engine(blp, comm=comm)
        sub_start = None
        if start is not None:
            y0 = np.broadcast_to(np.asarray(start[1], dtype=np.float64), (csr.shape[0],))
            sub_start = (start[0], y0[blk.rows], start[2])

        def run(cfg, t_start):
            x, yb, z, st, recs = eng.solve_raw(cfg, sub_start, time.perf_counter() - t_start,
                                               rows=blk.rows, m_total=csr.shape[0])
            parts = [None] * comm.world_size
            dist.all_gather_object(parts, (blk.rows, yb), group=group)
            y = np.empty(csr.shape[0])
            for rows, yy in parts:
                y[rows] = yy
            stats = {"loop_seconds": st.loop_seconds, "gpu_launches": int(st.gpu_launches),
                     "world_size": comm.world_size, "block_rows": int(blk.rows.size),
                     "block_nnz": int(blk.nnz)}
            return _assemble(lp, cfg, x, y, z, st, recs, t_start, stats)

        try:
            return _with_fp64_retry(config or SolverConfig(), run)
        finally:
            eng.close()
    finally:
        if own:
            comm.close()


# ---------------------------------------------------------------------------
# plug-in point
# ---------------------------------------------------------------------------

_SAVED = {}


_PRESOLVE_SITES = ("scuckit.presolve", "scuckit.fixing", "scuckit.milp_bb", "scuckit")


_SCREEN_SITES = ("scuckit.driver", "scuckit")


# where the reference imported the model builder / PTDF by name
_BUILDER_SITES = {"build_model": ("scuckit.formulation", "scuckit.driver", "scuckit"),
                  "compute_ptdf": ("scuckit.instance", "scuckit.formulation", "scuckit.driver",
                                   "scuckit")}


def install(module=None, presolve: bool = True, screen: bool = True, builder: bool = True,
            bb: bool = False):
    """Route the reference's LP solves to the GPU engine.

    Rebinds ``scuckit.hprlp.solve`` (and ``kkt_residual`` / ``hpr_iterate``)
    and switches result construction to the reference's own classes.  With
    ``presolve`` the reference's ``milp_presolve`` / ``lp_presolve`` are
    rebound too, in every module that imported them by name (presolve.py,
    fixing.py:22, milp_bb.py:26, the package namespace), to the native-core
    mirror in ``paper_2510_10891_b200.presolve`` (bit-identical reductions).
    With ``screen`` the driver's post-MILP flow screen
    (``driver.screen_violations``, ``driver.py:165-200``, called by name at
    ``:288``) is rebound to the device screen in ``screen.py``.  With
    ``builder`` the model construction the driver runs every filtering pass
    (``build_model``, ``driver.py:249-250``; ``compute_ptdf``, ``:210``) is
    rebound to ``builder.py``: the reference's own model objects, built
    vectorised (identical rows, bounds and tags), PTDF tables from one solve
    plus LODF updates.  With ``bb`` (opt-in) the branch-and-bound's
    ``_Search`` (``milp_bb.py:101-404``) solves a plunge's waiting sibling
    ahead on a second engine and stream (``bb.py``); every node result, hence
    the search, is unchanged.  It pays when dives are short and siblings are
    revisited, and costs GPU time a long dive needs."""
    import importlib
    if module is None:
        import scuckit.hprlp as module
    from scuckit import lp_kernel
    if "solve" not in _SAVED:
        _SAVED.update(solve=module.solve, kkt_residual=module.kkt_residual,
                      hpr_iterate=module.hpr_iterate, module=module, presolve={})
    _CLS.status = module.SolveStatus
    _CLS.result = module.SolveResult
    _CLS.kkt = module.KktResidual
    _CLS.precision = lp_kernel.Precision
    module.solve = solve
    module.kkt_residual = kkt_residual
    module.hpr_iterate = hpr_iterate
    if presolve:
        from . import presolve as native
        ref = importlib.import_module("scuckit.presolve")
        native._LOG_CLASS = ref.ReductionLog
        for name in _PRESOLVE_SITES:
            mod = importlib.import_module(name)
            for fn in ("milp_presolve", "lp_presolve"):
                if hasattr(mod, fn):
                    _SAVED["presolve"].setdefault((name, fn), getattr(mod, fn))
                    setattr(mod, fn, getattr(native, fn))
    if screen:
        from . import screen as dev_screen
        drv = importlib.import_module("scuckit.driver")
        dev_screen._VIOLATION_CLASS = drv.Violation
        for name in _SCREEN_SITES:
            mod = importlib.import_module(name)
            if hasattr(mod, "screen_violations"):
                _SAVED.setdefault("screen", {}).setdefault(name, mod.screen_violations)
                mod.screen_violations = dev_screen.screen_violations
    if bb:
        from . import bb as spec
        mbb = importlib.import_module("scuckit.milp_bb")
        lpb = importlib.import_module("scuckit.lp_backends")
        if "bb" not in _SAVED:
            _SAVED["bb"] = (mbb._Search, lpb.solve_lp)
        mbb._Search = spec.make_search_class(mbb, lpb)
        if getattr(lpb.solve_lp, "__wrapped__", None) is None:
            lpb.solve_lp = spec.wrap_solve_lp(lpb.solve_lp)
    if builder:
        from . import builder as fast
        for fn, sites in _BUILDER_SITES.items():
            for name in sites:
                mod = importlib.import_module(name)
                if hasattr(mod, fn):
                    _SAVED.setdefault("builder", {}).setdefault((name, fn), getattr(mod, fn))
                    setattr(mod, fn, getattr(fast, fn))
    return module


def uninstall():
    if not _SAVED:
        return
    import importlib
    module = _SAVED["module"]
    module.solve = _SAVED["solve"]
    module.kkt_residual = _SAVED["kkt_residual"]
    module.hpr_iterate = _SAVED["hpr_iterate"]
    for (name, fn), orig in _SAVED.get("presolve", {}).items():
        setattr(importlib.import_module(name), fn, orig)
    for name, orig in _SAVED.get("screen", {}).items():
        importlib.import_module(name).screen_violations = orig
    for (name, fn), orig in _SAVED.get("builder", {}).items():
        setattr(importlib.import_module(name), fn, orig)
    if "bb" in _SAVED:
        search, solve_lp = _SAVED["bb"]
        importlib.import_module("scuckit.milp_bb")._Search = search
        importlib.import_module("scuckit.lp_backends").solve_lp = solve_lp
    from . import presolve as native
    native._LOG_CLASS = native.ReductionLog
    from . import screen as dev_screen
    dev_screen._VIOLATION_CLASS = dev_screen.Violation
    _CLS.status, _CLS.result, _CLS.kkt, _CLS.precision = (SolveStatus, SolveResult,
                                                          KktResidual, Precision)
    _SAVED.clear()
