"""Device flow screen: mirror of ``scuckit.driver.screen_violations``.

Reference: ``pkg/src/scuckit/driver.py:165-200``.  After each MILP pass the
driver checks the unscaled point against every (line, period, contingency):
net injections per bus and period are rebuilt from the point
(``driver.py:176-181``), flows are ``ptdf.table(key) @ injections`` for every
key (``:185-186``) and a triple is reported when
``|flow| - limit > tol * limit`` (``:187-196``), sorted by excess, largest
first (``:199``).

Here the injections are rebuilt on the host exactly as the reference builds
them (same numpy operations in the same order, so bit-identical), and the
products plus the threshold test run on the GPU (``csrc/hpr_screen.cu``,
C-ABI ``include/hpr_screen.h``) against PTDF tables that stay resident in HBM
for the lifetime of the (immutable) ``PtdfTable``.  The FP64 sums are taken
in a different order than the host BLAS, so flows agree to rounding
(~1e-15 relative), and the violation set is the reference's except for
entries within rounding of the threshold.

There is no CPU fallback: without the library or a CUDA device the first
screen raises.
"""

from __future__ import annotations

import ctypes as C
import types
import weakref
from dataclasses import dataclass

import numpy as np

from . import _capi


@dataclass
class Violation:
    """Mirror of ``scuckit.driver.Violation`` (``driver.py:68-81``);
    ``install()`` switches results to the reference's own class."""
    line: str
    period: int
    contingency: str
    flow: float
    limit: float
    excess: float
    already_monitored: bool = False

    @property
    def triple(self) -> tuple:
        return (self.line, self.period, self.contingency)


_VIOLATION_CLASS = Violation
PERIODS_PER_LAUNCH = 96   # hpr_screen_run's limit (2 warp rows x 6 period tiles of 8)


def column_blocks(instance):
    """The columns ``screen_violations`` reads, as ``VariableMap`` lays them
    out (``formulation.py:42-70``): u at 0, p' at 3GT, then the segment
    columns (T * H_g per unit), the cost block (GT) and the unserved-demand
    block (B x T).  Returns (u, pprime, penalty, n_cols)."""
    n_g = len(instance.generators)
    n_t = instance.n_periods
    n_b = len(instance.buses)
    gt = n_g * n_t
    u = np.arange(gt, dtype=np.int64).reshape(n_g, n_t)
    pprime = 3 * gt + u
    col = 4 * gt + n_t * sum(g.n_segments for g in instance.generators) + gt
    penalty = col + np.arange(n_b * n_t, dtype=np.int64).reshape(n_b, n_t)
    return u, pprime, penalty, col + n_b * n_t


def injections(point, instance) -> np.ndarray:
    """Net injections (n_buses x n_periods), ``driver.py:176-181``."""
    u, pprime, penalty, n_cols = column_blocks(instance)
    point = np.asarray(point, dtype=np.float64)
    if point.shape[0] != n_cols:
        raise ValueError("point length does not match the instance's model")
    demand = instance.demand_matrix()
    bus_idx = instance.network.bus_index()
    power = point[pprime] + np.array([[g.p_min] for g in instance.generators]) * point[u]
    inj = -(demand - point[penalty])
    rows = np.array([bus_idx[g.bus] for g in instance.generators], dtype=np.int64)
    # unbuffered, in generator order: the same sequence of adds as the
    # reference's per-generator loop (driver.py:180-181)
    np.add.at(inj, rows, power)
    return inj


def _ranks(ids) -> np.ndarray:
    """Position of each id in Python string order (the sort key's tie-breaks)."""
    r = np.empty(len(ids), np.int64)
    r[sorted(range(len(ids)), key=ids.__getitem__)] = np.arange(len(ids))
    return r


class FlowScreen:
    """PTDF tables of one ``PtdfTable`` resident on one GPU, with the per-key
    line limits (``Line.limit_for``, ``instance.py:88-89``)."""

    def __init__(self, ptdf, keys, lines, device: int = 0):
        self.lib = _capi.load()
        self.device = int(device)
        self.keys = list(keys)
        self.line_ids = [ln.lid for ln in lines]
        tabs = [np.ascontiguousarray(ptdf.table(k), dtype=np.float64) for k in self.keys]
        n_l, n_b = tabs[0].shape
        if n_l != len(self.line_ids):
            raise ValueError("PTDF rows do not match the instance's lines")
        self.limits = limit_table(types.SimpleNamespace(lines=lines), self.keys)
        self.shape = (n_l, n_b)
        self.line_rank = _ranks(self.line_ids)
        self.key_rank = _ranks(self.keys)
        self._last_t = 0
        ptrs = (C.c_void_p * len(tabs))(*[t.ctypes.data for t in tabs])
        h = C.c_void_p()
        _capi.check(self.lib.hpr_screen_create(device, n_l, n_b, len(tabs), ptrs,
                                               _capi.ptr(self.limits), C.byref(h)))
        self.handle = h
        self._fin = weakref.finalize(self, self.lib.hpr_screen_destroy, h)

    def close(self):
        """Free the device tables; the object (and any cache entry holding
        it) is dead afterwards -- every later call raises."""
        self._fin()
        self.handle = None
        for key, ent in list(_SCREENS.items()):
            if ent[1] is self:
                _SCREENS.pop(key, None)

    def _h(self):
        if self.handle is None:
            raise ValueError("FlowScreen is closed")
        return self.handle

    def info(self) -> dict:
        info = _capi.ScreenInfo()
        _capi.check(self.lib.hpr_screen_info_get(self._h(), C.byref(info)))
        return {k: getattr(info, k) for k, _ in info._fields_}

    def run(self, inj: np.ndarray, tol: float):
        """Screen an (n_buses x n_periods) injection matrix; returns the
        records (table, line, period, flow, excess) as numpy arrays.  The
        kernel takes up to PERIODS_PER_LAUNCH periods; longer horizons run
        in period chunks (each (line, period) entry is independent)."""
        inj = np.ascontiguousarray(inj, dtype=np.float64)
        if inj.ndim != 2 or inj.shape[0] != self.shape[1]:
            raise ValueError("injections must be (n_buses, n_periods)")
        n_t = inj.shape[1]
        parts = []
        for t0 in range(0, max(n_t, 1), PERIODS_PER_LAUNCH):
            chunk = np.ascontiguousarray(inj[:, t0:t0 + PERIODS_PER_LAUNCH])
            n = C.c_int64()
            _capi.check(self.lib.hpr_screen_run(self._h(), _capi.ptr(chunk), chunk.shape[1],
                                                float(tol), C.byref(n)))
            k = n.value
            rec = (np.empty(k, np.int32), np.empty(k, np.int32), np.empty(k, np.int32),
                   np.empty(k, np.float64), np.empty(k, np.float64))
            _capi.check(self.lib.hpr_screen_fetch(self._h(), *[_capi.ptr(a) for a in rec]))
            rec[2][:] += t0
            parts.append(rec)
        self._last_t = n_t if n_t <= PERIODS_PER_LAUNCH else -1
        if len(parts) == 1:
            return parts[0]
        return tuple(np.concatenate([p[i] for p in parts]) for i in range(5))

    def flows(self, table: int = 0) -> np.ndarray:
        """Flows of one table from the last run (``PtdfTable.flows``,
        ``instance.py:170-173``)."""
        if self._last_t < 0:
            raise ValueError("flows() holds only the last period chunk of a long horizon")
        out = np.empty((self.shape[0], self._last_t), np.float64)
        _capi.check(self.lib.hpr_screen_flows(self._h(), table, _capi.ptr(out)))
        return out

    def bench(self, reps: int = 20) -> tuple:
        a, b = C.c_double(), C.c_double()
        _capi.check(self.lib.hpr_screen_bench(self._h(), reps, C.byref(a), C.byref(b)))
        return a.value, b.value


class _Line:
    __slots__ = ("lid", "limit", "emergency_limit")

    def __init__(self, d):
        self.lid, self.limit, self.emergency_limit = d["id"], d["limit"], d["emergency_limit"]

    def limit_for(self, key):                      # instance.py:88-89
        return self.limit if key == "base" else self.emergency_limit


def instance_view(doc: dict):
    """The attributes ``screen_violations`` reads from a ``ScucInstance``
    (``instance.py:99-139``), taken from a reference-schema instance document
    (for callers that hold the document but not a parsed instance)."""
    gens = tuple(types.SimpleNamespace(gid=g["id"], bus=g["bus"], p_min=g["p_min"],
                                       p_max=g["p_max"], n_segments=len(g["segments"]))
                 for g in doc["generators"])
    buses = tuple(types.SimpleNamespace(bid=b["id"], demand=b["demand"]) for b in doc["buses"])
    lines = tuple(_Line(ln) for ln in doc["lines"])
    conts = tuple(types.SimpleNamespace(cid=c["id"]) for c in doc.get("contingencies", ()))
    net = types.SimpleNamespace(buses=buses, lines=lines, contingencies=conts,
                                bus_index=lambda: {b.bid: i for i, b in enumerate(buses)})
    return types.SimpleNamespace(
        generators=gens, buses=buses, lines=lines, contingencies=conts, network=net,
        n_periods=doc["time_periods"],
        demand_matrix=lambda: np.array([b.demand for b in buses], dtype=np.float64),
        contingency_keys=lambda: ["base"] + [c.cid for c in conts])


class Tables:
    """``PtdfTable``'s read interface (``instance.py:166-168``) over a dict of
    (n_lines x n_buses) arrays keyed by contingency key."""

    def __init__(self, tables: dict):
        self._t = dict(tables)

    def keys(self) -> list:
        return list(self._t)

    def table(self, key: str = "base"):
        return self._t[key]


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured FP64 tensor-pipe ceiling (``hpr_fp64_peak_bench``)."""
    v = C.c_double()
    _capi.check(_capi.load().hpr_fp64_peak_bench(device, C.byref(v)))
    return v.value


_SCREENS: dict = {}


def limit_table(instance, keys) -> np.ndarray:
    """(len(keys) x n_lines) limits, ``Line.limit_for`` (instance.py:88-89):
    the normal limit for the base case, the emergency limit otherwise --
    one pass over the lines, then a broadcast over the keys."""
    lines = instance.lines
    base = np.array([ln.limit_for("base") for ln in lines], dtype=np.float64)
    cont = [k for k in keys if k != "base"]
    emer = (np.array([ln.limit_for(cont[0]) for ln in lines], dtype=np.float64)
            if cont else base)
    is_base = np.array([k == "base" for k in keys], dtype=bool)
    return np.ascontiguousarray(np.where(is_base[:, None], base[None, :], emer[None, :]))


def screen_for(ptdf, instance, device: int | None = None, keys=None) -> FlowScreen:
    """The resident screen of ``ptdf`` (built once; ``PtdfTable`` is
    immutable, ``instance.py:141-147``) on `device` (default: the caller's
    current CUDA device), rebuilt only if the device, the instance's keys or
    its limits differ from the ones it was built with.  ``keys`` restricts
    the resident tables to a subset of the instance's keys (one rank's
    shard)."""
    if device is None:
        import torch
        device = torch.cuda.current_device()
    keys = list(instance.contingency_keys() if keys is None else keys)
    ent = _SCREENS.get(id(ptdf))
    if ent is not None:
        ref, scr = ent
        if (ref() is ptdf and scr.handle is not None and scr.device == int(device)
                and scr.keys == keys and scr.line_ids == [ln.lid for ln in instance.lines]):
            if np.array_equal(limit_table(instance, keys), scr.limits):
                return scr
        scr.close()
    scr = FlowScreen(ptdf, keys, instance.lines, device=device)
    try:
        ref = weakref.ref(ptdf, lambda _r, key=id(ptdf): _drop(key))
    except TypeError:  # not weak-referenceable: keep it alive with the cache entry
        ref = (lambda obj: (lambda: obj))(ptdf)
    _SCREENS[id(ptdf)] = (ref, scr)
    return scr


def _drop(key):
    ent = _SCREENS.pop(key, None)
    if ent is not None:
        ent[1].close()


def _assemble(recs, keys, lids, lim, line_rank, key_rank, monitored) -> list:
    """Violation objects in the reference's order (driver.py:199): excess
    descending, then line id, period and contingency id as strings -- one
    lexsort over id ranks.  ``recs`` = (key index, line, period, flow, excess)."""
    tab, line, per, flow, exc = recs
    order = np.lexsort((key_rank[tab], per, line_rank[line], -exc))
    cls = _VIOLATION_CLASS
    tab, line, per = tab[order], line[order], per[order]
    cols = (tab.tolist(), line.tolist(), per.tolist(), flow[order].tolist(),
            lim[tab, line].tolist(), exc[order].tolist())
    if monitored:
        return [cls(lids[l], t, keys[k], f, li, e, (lids[l], t, keys[k]) in monitored)
                for k, l, t, f, li, e in zip(*cols)]
    return [cls(lids[l], t, keys[k], f, li, e, False) for k, l, t, f, li, e in zip(*cols)]


def screen_violations(point, instance, ptdf, monitored=(), tol: float = 1e-4) -> list:
    """Flow check of a primal vector over every (line, period, contingency);
    same signature, errors and result order as ``driver.py:165-200``."""
    inj = injections(point, instance)
    monitored = set(monitored)
    if len(instance.lines) == 0 or inj.shape[1] == 0:
        return []                     # nothing to screen (the reference's loops are empty)
    scr = screen_for(ptdf, instance)
    recs = scr.run(inj, tol)
    return _assemble(recs, scr.keys, scr.line_ids, scr.limits, scr.line_rank, scr.key_rank,
                     monitored)


def shard_keys(keys, world_size: int, rank: int) -> list:
    """The contingency keys one rank screens: round robin over the
    instance's key order (each key's product is independent, driver.py:184-186)."""
    return [k for i, k in enumerate(keys) if i % world_size == rank]


def screen_violations_sharded(point, instance, ptdf, monitored=(), tol: float = 1e-4,
                              group=None, device: int | None = None, _run=None) -> list:
    """``screen_violations`` with the contingency keys sharded over the ranks
    of a ``torch.distributed`` group, one GPU per rank (SURVEY §8(e) for the
    screen: independent products, so no data-path collective).  Each rank
    keeps only its shard's tables resident and screens them; the violation
    records are all-gathered once and every rank returns the same list, in
    the reference's order.  ``_run(keys, inj, tol)`` replaces the device
    screen of a shard (tests only)."""
    import torch.distributed as dist
    ws, rank = dist.get_world_size(group), dist.get_rank(group)
    inj = injections(point, instance)
    monitored = set(monitored)
    keys = list(instance.contingency_keys())
    if len(instance.lines) == 0 or inj.shape[1] == 0:
        return []
    mine = shard_keys(keys, ws, rank)
    if not mine:
        local = tuple(np.empty(0, t) for t in (np.int32, np.int32, np.int32, np.float64,
                                               np.float64))
    elif _run is not None:
        local = _run(mine, inj, tol)
    else:
        if device is None:
            import torch
            device = torch.cuda.current_device()
        local = screen_for(ptdf, instance, device=device, keys=mine).run(inj, tol)
    where = {k: i for i, k in enumerate(keys)}
    pos = np.array([where[k] for k in mine] or [0], dtype=np.int32)
    local = (pos[local[0]],) + tuple(local[1:])
    parts = [None] * ws
    dist.all_gather_object(parts, local, group=group)
    recs = tuple(np.concatenate([p[i] for p in parts]) for i in range(5))
    lids = [ln.lid for ln in instance.lines]
    return _assemble(recs, keys, lids, limit_table(instance, keys), _ranks(lids), _ranks(keys),
                     monitored)
