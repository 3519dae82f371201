"""Synthetic SCUC instances and a vectorised LP-relaxation builder.

This module produces the LPs the HPR engine is measured on.  It has two
halves:

* ``generate_instance`` — a seeded generator that emits the reference's
  instance JSON schema (``scuckit/instance.py:358-461``), following the
  recipe in SURVEY.md §8(d): random spanning tree + chords, three equal-width
  cost segments, Dirichlet demand shares, pro-rata-dispatch line limits.
* ``build_relaxation`` — a numpy restatement of ``build_model`` +
  ``MilpModel.relax`` (``scuckit/formulation.py:215-413``, ``:143-145``)
  that emits the same standard-form LP (CSR arrays, rhs, cost, bounds,
  ``n_eq``) without the per-entry Python loop, so 13,659-bus LPs with
  tens of millions of nonzeros build in seconds.  It reproduces the
  reference's floating-point operations term by term, and the test suite
  checks it is CSR-identical to the reference builder on small instances.

Column layout follows ``VariableMap`` (``formulation.py:35-80``): u, v, w,
p' blocks [g, t], per-generator segment blocks [t, h], cost [g, t],
unserved-demand slacks [b, t].  Row order follows ``build_model``: the
equality block (logic, segment sum, cost definition, balance) then the
inequality block (logic, min-up, min-down, production limit, ramp-up,
ramp-down, segment caps, flow lo/hi pairs for sorted monitored triples).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

BASE_CASE = "base"
_FLOW_COEFF_DROP = 1e-10          # formulation.py:23


# ---------------------------------------------------------------------------
# instance generation
# ---------------------------------------------------------------------------

# Named configurations of BASELINE.json "configs" (sizes from SURVEY.md §8(d)).
CONFIGS = {
    "C1": dict(n_buses=118, n_gens=54, n_lines=186, n_periods=24, seed=1),
    "C2": dict(n_buses=1354, n_gens=260, n_lines=1991, n_periods=24, seed=2),
    "C3": dict(n_buses=6468, n_gens=399, n_lines=9000, n_periods=36, seed=3),
    "C4": dict(n_buses=13659, n_gens=4092, n_lines=20467, n_periods=36, seed=4),
    # C4 plus 64 single-line (chord) outages; monitors 20,000 N-1 (line, period,
    # contingency) triples -> ~874M nonzeros (BASELINE configs[4])
    "C5": dict(n_buses=13659, n_gens=4092, n_lines=20467, n_periods=36, seed=4,
               n_contingencies=64),
}


def _r(x, nd):
    """Round generated data so the instance is robust to last-bit noise in
    the linear solves used to derive it (instances are data, not results)."""
    return np.round(np.asarray(x, dtype=np.float64), nd)


def _bus_laplacian_reduced(n_b, fb, tb, react, ref=0):
    import scipy.sparse as sp
    b = 1.0 / react
    rows = np.concatenate([fb, tb, fb, tb])
    cols = np.concatenate([fb, tb, tb, fb])
    vals = np.concatenate([b, b, -b, -b])
    lap = sp.csc_matrix((vals, (rows, cols)), shape=(n_b, n_b))
    keep = np.flatnonzero(np.arange(n_b) != ref)
    return lap[keep][:, keep].tocsc(), keep


def _dc_flows(n_b, fb, tb, react, injections, ref=0):
    """Line flows (L x T) of bus injections (B x T) under the DC model, by a
    sparse solve of the reference-reduced susceptance system."""
    import scipy.sparse.linalg as spla
    lap, keep = _bus_laplacian_reduced(n_b, fb, tb, react, ref)
    theta = np.zeros((n_b, injections.shape[1]))
    rhs = np.ascontiguousarray(injections[keep])
    if n_b <= 2000:
        theta[keep] = spla.splu(lap).solve(rhs)
    else:
        # random chords make sparse LU fill in; the reduced Laplacian is SPD,
        # so Jacobi-preconditioned CG is cheap (limits are rounded to 1e-3 MW)
        lap = lap.tocsr()
        dinv = 1.0 / lap.diagonal()
        pre = spla.LinearOperator(lap.shape, matvec=lambda v: dinv * v)
        for k in range(rhs.shape[1]):
            sol, info = spla.cg(lap, rhs[:, k], rtol=1e-13, atol=0.0, maxiter=20000, M=pre)
            if info != 0:
                raise RuntimeError("DC-flow CG did not converge")
            theta[keep, k] = sol
    return (theta[fb] - theta[tb]) / react[:, None]


def generate_instance(n_buses: int, n_gens: int, n_lines: int, n_periods: int,
                      seed: int = 0, n_contingencies: int = 0,
                      name: str | None = None, shutdown_feasible: bool = False) -> dict:
    """Seeded synthetic SCUC instance as a reference-schema JSON document.

    shutdown_feasible caps every committed unit's initial output at its
    shutdown limit, so switching it off in period 0 stays feasible (the
    ramp-down row at t = 0, formulation.py:331-341); without it, rounding a
    fractional u_0 to 0 can make the fixed model infeasible, which aborts the
    reference driver (fixing.py:154-160).  The default keeps the fixtures'
    instances unchanged."""
    if n_lines < n_buses - 1:
        raise ValueError("need at least n_buses - 1 lines for a connected network")
    rng = np.random.default_rng(seed)
    B, G, L, T = n_buses, n_gens, n_lines, n_periods

    # network: random spanning tree (each bus attaches to an earlier one) + chords
    parent = np.array([rng.integers(0, i) for i in range(1, B)], dtype=np.int64)
    fb = np.concatenate([parent, np.zeros(0, np.int64)])
    tb = np.arange(1, B, dtype=np.int64)
    n_ch = L - (B - 1)
    ci = rng.integers(0, B, size=n_ch)
    cj = (ci + rng.integers(1, B, size=n_ch)) % B      # cj != ci
    fb = np.concatenate([fb, ci]).astype(np.int64)
    tb = np.concatenate([tb, cj]).astype(np.int64)
    react = _r(rng.uniform(0.01, 0.1, size=L), 5)

    # generators
    gbus = rng.integers(0, B, size=G)
    pmax = _r(rng.uniform(50.0, 500.0, size=G), 3)
    pmin = _r(pmax * rng.uniform(0.2, 0.5, size=G), 3)
    c0 = _r(rng.uniform(10.0, 60.0, size=G), 4)
    ut = rng.integers(1, 9, size=G)
    dt = rng.integers(1, 9, size=G)
    on = (rng.uniform(size=G) < 0.6).astype(np.int64)
    init_frac = rng.uniform(size=G)
    init_per = rng.integers(1, 9, size=G)

    # demand: Dirichlet shares x (0.55 + 0.15 sin) x total capacity
    shares = rng.dirichlet(np.ones(B))
    prof = 0.55 + 0.15 * np.sin(2.0 * np.pi * np.arange(T) / T)
    total = prof * pmax.sum()
    demand = _r(np.outer(shares, total), 4)

    # line limits from the DC flows of a pro-rata dispatch
    frac = demand.sum(axis=0) / pmax.sum()
    inj = -demand.copy()
    np.add.at(inj, gbus, np.outer(pmax, frac))
    flows = _dc_flows(B, fb, tb, react, inj)
    peak = np.abs(flows).max(axis=1)
    congested = rng.uniform(size=L) < 0.1
    limit = _r(np.maximum(np.where(congested, 0.9, 2.0) * peak, 1.0), 3)

    gens = []
    for g in range(G):
        lo, hi = float(pmin[g]), float(pmax[g])
        w3 = (hi - lo) / 3.0
        caps = [round(lo + w3, 6), round(lo + 2.0 * w3, 6), hi]
        if not (lo < caps[0] < caps[1] < caps[2]):
            caps = [hi]
        cst = [float(c0[g]) * f for f in (1.0, 1.15, 1.3)][: len(caps)]
        su = max(lo, round(0.6 * hi, 3))
        ip = round(lo + init_frac[g] * 0.5 * (hi - lo), 3) if on[g] else 0.0
        if shutdown_feasible:
            ip = min(ip, su)
        gens.append({
            "id": f"g{g}", "bus": f"b{int(gbus[g])}", "p_min": lo, "p_max": hi,
            "segments": [{"p_max": c, "cost": round(k, 6)} for c, k in zip(caps, cst)],
            "min_output_cost": round(float(c0[g]) * lo, 4),
            "min_up": int(ut[g]), "min_down": int(dt[g]),
            "ramp_up": round(0.5 * hi, 3), "ramp_down": round(0.5 * hi, 3),
            "startup_limit": su, "shutdown_limit": su,
            "initial_on": int(on[g]), "initial_power": ip,
            "initial_periods": int(init_per[g]),
        })

    conts = []
    if n_contingencies:
        # outage candidates: chords only (tree edges are bridges of the tree
        # but chords keep every bus connected when one chord is removed)
        cand = np.arange(B - 1, L)
        pick = rng.choice(cand, size=min(n_contingencies, cand.size), replace=False)
        conts = [{"id": f"c{int(k)}", "line": f"l{int(k)}"} for k in np.sort(pick)]

    return {
        "name": name or f"synthetic-{B}b-{G}g-{T}t-s{seed}",
        "time_periods": int(T),
        "penalty_cost": 1000.0,
        "reference_bus": "b0",
        "buses": [{"id": f"b{b}", "demand": demand[b].tolist()} for b in range(B)],
        "lines": [{"id": f"l{k}", "from": f"b{int(fb[k])}", "to": f"b{int(tb[k])}",
                   "reactance": float(react[k]), "limit": float(limit[k]),
                   "emergency_limit": float(_r(1.2 * limit[k], 3))} for k in range(L)],
        "contingencies": conts,
        "generators": gens,
    }


def sample_monitored(doc: dict, n_triples: int, seed: int = 0,
                     contingencies: bool = False) -> list:
    """Seeded uniform draw of distinct (line_id, period, key) triples."""
    rng = np.random.default_rng(seed + 7919)
    L = len(doc["lines"])
    T = doc["time_periods"]
    keys = [BASE_CASE]
    if contingencies:
        keys = [c["id"] for c in doc["contingencies"]]
    total = L * T * len(keys)
    n = min(n_triples, total)
    flat = rng.choice(total, size=n, replace=False)
    out = []
    for f in flat:
        k, rem = divmod(int(f), L * T)
        l, t = divmod(rem, T)
        out.append((doc["lines"][l]["id"], t, keys[k]))
    return out


def all_base_triples(doc: dict) -> list:
    return [(ln["id"], t, BASE_CASE) for ln in doc["lines"] for t in range(doc["time_periods"])]


# ---------------------------------------------------------------------------
# standard-form LP container (mirrors scuckit.lp_kernel.StandardFormLp)
# ---------------------------------------------------------------------------

@dataclass
class LpArrays:
    """Standard-form LP  min cost.x + offset  s.t.  A x (= first n_eq | >=) rhs,
    lower <= x <= upper, as plain arrays (CSR int32 indptr/indices, f64 data)."""

    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    shape: tuple
    rhs: np.ndarray
    cost: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    n_eq: int
    offset: float = 0.0

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def csr(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.data, self.indices, self.indptr), shape=self.shape)

    def digest(self) -> str:
        import hashlib
        h = hashlib.sha256()
        for a in (self.indptr.astype(np.int64), self.indices.astype(np.int64), self.data,
                  self.rhs, self.cost, self.lower, self.upper):
            h.update(np.ascontiguousarray(a).tobytes())
        h.update(f"{self.shape}{self.n_eq}{self.offset!r}".encode())
        return h.hexdigest()

    def digest_parts(self) -> dict:
        """Per-array digests (which part of two LPs differs)."""
        import hashlib
        return {k: hashlib.sha256(np.ascontiguousarray(getattr(self, k)).tobytes()).hexdigest()[:16]
                for k in ("indptr", "indices", "data", "rhs", "cost", "lower", "upper")}

    def to_lp(self):
        """As a duck-typed StandardFormLp (``.matrix.csr/.csc``, vectors)."""
        from .lp import StandardFormLp, SparseMatrix
        return StandardFormLp(matrix=SparseMatrix.from_csr_arrays(
            self.indptr, self.indices, self.data, self.shape),
            rhs=self.rhs, cost=self.cost, lower=self.lower, upper=self.upper,
            n_eq=self.n_eq, offset=self.offset)


# ---------------------------------------------------------------------------
# PTDF rows
# ---------------------------------------------------------------------------

# Host PTDF solves run under a fixed-size BLAS thread pool.  OpenBLAS splits a
# dense solve by thread count, so its last bits depend on it: with the pool
# pinned, the build container (8 cores) and the B200 box (16 cores, same CPU
# model) produce bit-identical PTDF rows, hence identical LPs (digests), which
# is what lets the committed reference trajectories be replayed on the box.
PTDF_BLAS_THREADS = 8
# ...and every other BLAS call of a named-config build (the flow rows' base
# dot products, 13,659-long at C4, are threaded by OpenBLAS above 10^4
# entries) under a pool of this size
BUILD_BLAS_THREADS = 2


def _blas_pool(n=None):
    from threadpoolctl import threadpool_limits
    return threadpool_limits(PTDF_BLAS_THREADS if n is None else n)


def _ptdf_full_reference(n_b, fb, tb, react, ref, skip=None):
    """PTDF exactly as ``instance._ptdf_matrix`` computes it
    (``scuckit/instance.py:199-238``): dense solve of the reduced B-matrix
    against the identity, row differences divided by reactance."""
    import scipy.linalg
    b_full = np.zeros((n_b, n_b))
    for k in range(len(fb)):
        if k == skip:
            continue
        i, j = fb[k], tb[k]
        b = 1.0 / react[k]
        b_full[i, i] += b
        b_full[j, j] += b
        b_full[i, j] -= b
        b_full[j, i] -= b
    keep = [i for i in range(n_b) if i != ref]
    b_red = b_full[np.ix_(keep, keep)]
    with _blas_pool():
        theta_red = scipy.linalg.solve(b_red, np.eye(n_b - 1), assume_a="sym")
    theta = np.zeros((n_b, n_b))
    theta[np.ix_(keep, keep)] = theta_red
    delta = np.zeros((len(fb), n_b))
    for k in range(len(fb)):
        if k == skip:
            continue
        delta[k, :] = (theta[fb[k], :] - theta[tb[k], :]) / react[k]
    delta[:, ref] = 0.0
    return delta


def _ptdf_rows_direct(n_b, fb, tb, react, ref, lines, skip=None, device=None):
    """PTDF rows of `lines` only: solve B_red W = E for the line incidence
    columns (dense LU; on a CUDA device through torch when one is given).
    Agrees with the reference table to rounding, not bit-for-bit."""
    keep = np.flatnonzero(np.arange(n_b) != ref)
    pos = np.full(n_b, -1, np.int64)
    pos[keep] = np.arange(keep.size)
    mask = np.ones(len(fb), bool)
    if skip is not None:
        mask[skip] = False
    b = 1.0 / react[mask]
    f, t = fb[mask], tb[mask]
    nk = keep.size
    if device is not None:
        import torch
        dev = torch.device(device)
        bred = torch.zeros((n_b, n_b), dtype=torch.float64, device=dev)
        fi = torch.as_tensor(f, device=dev)
        ti = torch.as_tensor(t, device=dev)
        bb = torch.as_tensor(b, device=dev)
        bred.index_put_((fi, fi), bb, accumulate=True)
        bred.index_put_((ti, ti), bb, accumulate=True)
        bred.index_put_((fi, ti), -bb, accumulate=True)
        bred.index_put_((ti, fi), -bb, accumulate=True)
        kk = torch.as_tensor(keep, device=dev)
        bred = bred[kk][:, kk]
        rhs = torch.zeros((nk, len(lines)), dtype=torch.float64, device=dev)
        for c, k in enumerate(lines):
            if pos[fb[k]] >= 0:
                rhs[pos[fb[k]], c] += 1.0
            if pos[tb[k]] >= 0:
                rhs[pos[tb[k]], c] -= 1.0
        w = torch.linalg.solve(bred, rhs).cpu().numpy()
        del bred, rhs
    else:
        import scipy.linalg
        bred = np.zeros((n_b, n_b))
        np.add.at(bred, (f, f), b)
        np.add.at(bred, (t, t), b)
        np.add.at(bred, (f, t), -b)
        np.add.at(bred, (t, f), -b)
        bred = bred[np.ix_(keep, keep)]
        rhs = np.zeros((nk, len(lines)))
        for c, k in enumerate(lines):
            if pos[fb[k]] >= 0:
                rhs[pos[fb[k]], c] += 1.0
            if pos[tb[k]] >= 0:
                rhs[pos[tb[k]], c] -= 1.0
        with _blas_pool():
            w = scipy.linalg.solve(bred, rhs, assume_a="sym")
    out = np.zeros((len(lines), n_b))
    out[:, keep] = w.T
    out /= react[np.asarray(lines)][:, None]
    if skip is not None:
        out[np.asarray(lines) == skip] = 0.0
    out[:, ref] = 0.0
    return out


def _lodf_rows(base: np.ndarray, base_pk: np.ndarray, lines, k: int, fb, tb, ref: int):
    """Post-contingency PTDF rows by the line-outage distribution factor
    (LODF) update instead of a fresh factorisation per contingency
    (``compute_ptdf`` refactorises, ``instance.py:241-267``): with line k
    (f -> t) out,

        PTDF_c[l, :] = PTDF[l, :] + LODF[l, k] * PTDF[k, :],
        LODF[l, k]   = (PTDF[l, f] - PTDF[l, t]) / (1 - (PTDF[k, f] - PTDF[k, t])),

    the outaged line's own row is zero and the reference-bus column stays
    zero, as ``_ptdf_matrix(skip_line=k)`` leaves them (``instance.py:230-238``).
    Equal to the refactorised table to rounding (tests/test_builder.py)."""
    f, t = int(fb[k]), int(tb[k])
    den = 1.0 - (base_pk[f] - base_pk[t])
    num = base[:, f] - base[:, t]
    out = base + (num / den)[:, None] * base_pk[None, :]
    out[np.asarray(lines) == k] = 0.0
    out[:, ref] = 0.0
    return out


class PtdfRows:
    """Lazy PTDF row provider: ``row(line_pos, key)``.

    ``method="reference"`` reproduces ``compute_ptdf``'s dense tables bit for
    bit (small networks); ``"direct"`` solves only for the needed rows
    (optionally on a CUDA device), which is what 13,659-bus instances need —
    ``build_model`` only ever indexes ``ptdf.table(key)[row, :]``
    (``formulation.py:354``).  ``"lodf"`` takes the base rows as "direct" does
    and derives every contingency row from them by the LODF update (one
    solve for all N-1 keys: what the C5 instances need)."""

    def __init__(self, net, method="reference", device=None, needed=None):
        self.net = net
        self.method = method
        self.device = device
        self._tables = {}
        self._rows = {}
        self._base = {}
        self._needed = needed or {}

    def _base_rows(self, lines):
        net = self.net
        missing = sorted({int(q) for q in lines} - set(self._base))
        if missing:
            rows = _ptdf_rows_direct(net.n_b, net.fb, net.tb, net.react, net.ref, missing,
                                     device=self.device)
            for c, q in enumerate(missing):
                self._base[q] = rows[c]
        return np.stack([self._base[int(q)] for q in lines]) if len(lines) else \
            np.zeros((0, net.n_b))

    def row(self, lpos: int, key: str) -> np.ndarray:
        net = self.net
        skip = None if key == BASE_CASE else net.cont_line[key]
        if self.method == "lodf":
            if (lpos, key) not in self._rows:
                if not self._base:
                    # one solve for every base row any key needs (lines + outages)
                    want = set()
                    for kk, ls in self._needed.items():
                        want |= set(ls)
                        if kk != BASE_CASE:
                            want.add(net.cont_line[kk])
                    self._base_rows(sorted(want | {lpos}))
                lines = sorted(set(self._needed.get(key, [])) | {lpos})
                base = self._base_rows(lines)
                if key == BASE_CASE:
                    rows = base
                else:
                    rows = _lodf_rows(base, self._base_rows([skip])[0], lines, skip,
                                      net.fb, net.tb, net.ref)
                for c, q in enumerate(lines):
                    self._rows[(q, key)] = rows[c]
            return self._rows[(lpos, key)]
        if self.method == "reference":
            if key not in self._tables:
                self._tables[key] = _ptdf_full_reference(
                    net.n_b, net.fb, net.tb, net.react, net.ref, skip)
            return self._tables[key][lpos]
        if (lpos, key) not in self._rows:
            lines = sorted(set(self._needed.get(key, [])) | {lpos})
            rows = _ptdf_rows_direct(net.n_b, net.fb, net.tb, net.react, net.ref,
                                     lines, skip=skip, device=self.device)
            for c, k in enumerate(lines):
                self._rows[(k, key)] = rows[c]
        return self._rows[(lpos, key)]


# ---------------------------------------------------------------------------
# parsed instance (arrays) — mirrors the fields build_model reads
# ---------------------------------------------------------------------------

@dataclass
class _Net:
    n_b: int
    fb: np.ndarray
    tb: np.ndarray
    react: np.ndarray
    ref: int
    cont_line: dict


class Instance:
    """Array view of a reference-schema instance document (the subset of
    ``parse_instance`` that ``build_model`` consumes; no validation beyond
    what indexing needs)."""

    def __init__(self, doc: dict):
        self.doc = doc
        self.T = int(doc["time_periods"])
        self.penalty = float(doc["penalty_cost"])
        buses = doc["buses"]
        self.bus_ids = [str(b["id"]) for b in buses]
        bidx = {b: i for i, b in enumerate(self.bus_ids)}
        self.B = len(buses)
        self.demand = np.array([[float(d) for d in b["demand"]] for b in buses], dtype=np.float64)
        lines = doc.get("lines", [])
        self.line_ids = [str(l["id"]) for l in lines]
        self.line_pos = {l: i for i, l in enumerate(self.line_ids)}
        fb = np.array([bidx[str(l["from"])] for l in lines], dtype=np.int64)
        tb = np.array([bidx[str(l["to"])] for l in lines], dtype=np.int64)
        react = np.array([float(l["reactance"]) for l in lines], dtype=np.float64)
        self.limit = np.array([float(l["limit"]) for l in lines], dtype=np.float64)
        self.elimit = np.array([float(l.get("emergency_limit", l["limit"])) for l in lines],
                               dtype=np.float64)
        cont_line = {str(c["id"]): self.line_pos[str(c["line"])]
                     for c in doc.get("contingencies", [])}
        ref = bidx[str(doc.get("reference_bus", self.bus_ids[0]))]
        self.net = _Net(self.B, fb, tb, react, ref, cont_line)
        gens = doc["generators"]
        self.G = len(gens)
        self.gen_bus = np.array([bidx[str(g["bus"])] for g in gens], dtype=np.int64)
        f = lambda k: np.array([float(g[k]) for g in gens], dtype=np.float64)
        self.pmin, self.pmax = f("p_min"), f("p_max")
        self.min_cost = f("min_output_cost")
        self.ru, self.rd = f("ramp_up"), f("ramp_down")
        self.su, self.sd = f("startup_limit"), f("shutdown_limit")
        self.init_power = f("initial_power")
        self.init_on = np.array([int(g["initial_on"]) for g in gens], dtype=np.int64)
        self.init_per = np.array([int(g["initial_periods"]) for g in gens], dtype=np.int64)
        self.min_up = np.array([int(g["min_up"]) for g in gens], dtype=np.int64)
        self.min_down = np.array([int(g["min_down"]) for g in gens], dtype=np.int64)
        self.seg_caps = [[float(s["p_max"]) for s in g["segments"]] for g in gens]
        self.seg_costs = [[float(s["cost"]) for s in g["segments"]] for g in gens]
        self.H = np.array([len(c) for c in self.seg_caps], dtype=np.int64)

    @classmethod
    def from_scuckit(cls, inst) -> "Instance":
        """The same array view of a parsed (and possibly instance-scaled)
        reference ``ScucInstance`` (``instance.py:29-139``,
        ``formulation.apply_instance_scaling`` :148-191): what the drop-in
        ``build_model`` reads, so scaled MW / $ values reach the rows exactly
        as the reference's generator and bus attributes carry them."""
        self = cls.__new__(cls)
        self.doc = None
        net = inst.network
        self.T = int(inst.n_periods)
        self.penalty = float(inst.penalty_cost)
        self.bus_ids = [b.bid for b in net.buses]
        bidx = net.bus_index()
        self.B = len(net.buses)
        self.demand = inst.demand_matrix()
        lines = net.lines
        self.line_ids = [ln.lid for ln in lines]
        self.line_pos = net.line_index()
        fb = np.array([bidx[ln.from_bus] for ln in lines], dtype=np.int64)
        tb = np.array([bidx[ln.to_bus] for ln in lines], dtype=np.int64)
        react = np.array([ln.reactance for ln in lines], dtype=np.float64)
        self.limit = np.array([ln.limit for ln in lines], dtype=np.float64)
        self.elimit = np.array([ln.emergency_limit for ln in lines], dtype=np.float64)
        cont_line = {c.cid: self.line_pos[c.line] for c in net.contingencies}
        self.net = _Net(self.B, fb, tb, react, bidx[net.reference_bus], cont_line)
        gens = inst.generators
        self.G = len(gens)
        self.gen_bus = np.array([bidx[g.bus] for g in gens], dtype=np.int64)
        f = lambda k: np.array([float(getattr(g, k)) for g in gens], dtype=np.float64)  # noqa: E731
        self.pmin, self.pmax = f("p_min"), f("p_max")
        self.min_cost = f("min_output_cost")
        self.ru, self.rd = f("ramp_up"), f("ramp_down")
        self.su, self.sd = f("startup_limit"), f("shutdown_limit")
        self.init_power = f("initial_power")
        self.init_on = np.array([int(g.initial_on) for g in gens], dtype=np.int64)
        self.init_per = np.array([int(g.initial_periods) for g in gens], dtype=np.int64)
        self.min_up = np.array([int(g.min_up) for g in gens], dtype=np.int64)
        self.min_down = np.array([int(g.min_down) for g in gens], dtype=np.int64)
        self.seg_caps = [[float(c) for c in g.segment_caps] for g in gens]
        self.seg_costs = [[float(c) for c in g.segment_costs] for g in gens]
        self.H = np.array([len(c) for c in self.seg_caps], dtype=np.int64)
        return self

    def widths(self, g):
        prev = float(self.pmin[g])
        out = []
        for cap in self.seg_caps[g]:
            out.append(cap - prev)
            prev = cap
        return out


# ---------------------------------------------------------------------------
# vectorised build_model + relax
# ---------------------------------------------------------------------------

class _Rows:
    """Accumulates row blocks as (row-local index, col, value) triples."""

    def __init__(self):
        self.r, self.c, self.v, self.rhs = [], [], [], []
        self.n = 0

    def block(self, n_rows, rr, cc, vv, theta):
        rr = np.asarray(rr, dtype=np.int64)
        vv = np.asarray(vv, dtype=np.float64)
        keep = vv != 0.0                  # add_row drops exact zeros (formulation.py:246)
        self.r.append(rr[keep] + self.n)
        self.c.append(np.asarray(cc, dtype=np.int64)[keep])
        self.v.append(vv[keep])
        self.rhs.append(np.broadcast_to(np.asarray(theta, dtype=np.float64), (n_rows,)).copy())
        self.n += n_rows


def build_relaxation(doc_or_inst, monitored=(), ptdf: PtdfRows | None = None,
                     ptdf_method: str = "reference", device=None) -> LpArrays:
    """LP relaxation of the SCUC MILP over `monitored` triples, identical to
    ``build_model(instance, monitored)[0].relax()`` (``formulation.py:215-413``)."""
    inst = doc_or_inst if isinstance(doc_or_inst, Instance) else Instance(doc_or_inst)
    G, T, B = inst.G, inst.T, inst.B
    GT = G * T
    g_of = np.repeat(np.arange(G), T)          # [g, t] flattening
    t_of = np.tile(np.arange(T), G)
    u = np.arange(GT, dtype=np.int64)
    v = u + GT
    w = u + 2 * GT
    pp = u + 3 * GT
    col = 4 * GT
    seg_base = np.zeros(G, dtype=np.int64)     # segments[g][t, h] = seg_base[g] + t*H + h
    for g in range(G):
        seg_base[g] = col
        col += T * int(inst.H[g])
    cst = col + u
    col += GT
    pen = col + np.arange(B * T, dtype=np.int64)   # penalty[b, t] = pen[b*T + t]
    n = col + B * T
    demand = inst.demand

    rows = _Rows()
    ar = np.arange(GT)

    # ---- equality block --------------------------------------------------
    # logic-eq: u_t - u_{t-1} - v_t + w_t = [u_0 at t=0]          (:254-263)
    t0 = t_of == 0
    rr = [ar, ar, ar, ar[~t0]]
    cc = [u, v, w, u[~t0] - 1]
    vv = [np.ones(GT), -np.ones(GT), np.ones(GT), -np.ones((~t0).sum())]
    theta = np.where(t0, inst.init_on[g_of].astype(np.float64), 0.0)
    rows.block(GT, np.concatenate(rr), np.concatenate(cc), np.concatenate(vv), theta)

    # seg-sum and cost-def                                         (:265-276)
    seg_r, seg_c, seg_h, seg_cost = [], [], [], []
    for g in range(G):
        Hg = int(inst.H[g])
        tt = np.repeat(np.arange(T), Hg)
        hh = np.tile(np.arange(Hg), T)
        seg_r.append(g * T + tt)
        seg_c.append(seg_base[g] + tt * Hg + hh)
        seg_h.append(hh)
        seg_cost.append(np.asarray(inst.seg_costs[g], dtype=np.float64)[hh])
    seg_r = np.concatenate(seg_r)
    seg_c = np.concatenate(seg_c)
    seg_cost = np.concatenate(seg_cost)
    rows.block(GT, np.concatenate([seg_r, ar]), np.concatenate([seg_c, pp]),
               np.concatenate([np.ones(seg_r.size), -np.ones(GT)]), 0.0)
    rows.block(GT, np.concatenate([seg_r, ar]), np.concatenate([seg_c, cst]),
               np.concatenate([seg_cost, -np.ones(GT)]), 0.0)

    # balance t                                                    (:278-285)
    bt_r = np.concatenate([t_of, t_of, np.tile(np.arange(T), B)])
    bt_c = np.concatenate([pp, u, pen])
    bt_v = np.concatenate([np.ones(GT), inst.pmin[g_of], np.ones(B * T)])
    bal_rhs = np.array([float(demand[:, t].sum()) for t in range(T)])
    rows.block(T, bt_r, bt_c, bt_v, bal_rhs)
    n_eq = rows.n

    # ---- inequality block -------------------------------------------------
    rows.block(GT, np.concatenate([ar, ar]), np.concatenate([v, w]),
               -np.ones(2 * GT), -1.0)                                   # logic-ineq

    def window_rows(main_col, main_val, win_cols, dur, theta):
        # u_t (+/-) and -x_tau for tau in [max(0, t-dur+1), t]         (:295-307)
        r_l, c_l, v_l = [ar], [main_col], [np.full(GT, main_val)]
        first = np.maximum(0, t_of - dur[g_of] + 1)
        for back in range(T):
            tau = t_of - back
            sel = tau >= first
            r_l.append(ar[sel])
            c_l.append(win_cols[sel] - back)
            v_l.append(-np.ones(sel.sum()))
        rows.block(GT, np.concatenate(r_l), np.concatenate(c_l), np.concatenate(v_l), theta)

    window_rows(u, 1.0, v, inst.min_up, 0.0)                             # min-up
    window_rows(u, -1.0, w, inst.min_down, -1.0)                         # min-down

    span = (inst.pmax - inst.pmin)[g_of]                                 # prod-limit
    rows.block(GT, np.concatenate([ar, ar]), np.concatenate([u, pp]),
               np.concatenate([span, -np.ones(GT)]), 0.0)

    pmin_g = inst.pmin[g_of]
    # ramp-up                                                            (:315-327)
    rr = [ar, ar, ar, ar[~t0], ar[~t0]]
    cc = [v, pp, u, u[~t0] - 1, pp[~t0] - 1]
    vv = [inst.su[g_of], -np.ones(GT), -pmin_g, (inst.ru + inst.pmin)[g_of][~t0],
          np.ones((~t0).sum())]
    theta = np.zeros(GT)
    theta[t0] = -(inst.ru * inst.init_on + inst.init_power)
    rows.block(GT, np.concatenate(rr), np.concatenate(cc), np.concatenate(vv), theta)
    # ramp-down                                                          (:329-341)
    rr = [ar, ar, ar, ar[~t0], ar[~t0]]
    cc = [u, w, pp, u[~t0] - 1, pp[~t0] - 1]
    vv = [(inst.rd + inst.pmin)[g_of], inst.sd[g_of], np.ones(GT), -pmin_g[~t0],
          -np.ones((~t0).sum())]
    theta = np.zeros(GT)
    theta[t0] = inst.init_power
    rows.block(GT, np.concatenate(rr), np.concatenate(cc), np.concatenate(vv), theta)

    # seg-cap (g, t, h)                                                  (:343-349)
    sc_r, sc_c, sc_v, off = [], [], [], 0
    seg_u, seg_col, seg_w = [], [], []
    for g in range(G):
        Hg = int(inst.H[g])
        wd = np.asarray(inst.widths(g), dtype=np.float64)
        k = np.arange(T * Hg)
        seg_u.append(g * T + k // Hg)
        seg_col.append(seg_base[g] + k)
        seg_w.append(wd[k % Hg])
    seg_u = np.concatenate(seg_u)
    seg_col = np.concatenate(seg_col)
    seg_w = np.concatenate(seg_w)
    ns = seg_u.size
    ars = np.arange(ns)
    rows.block(ns, np.concatenate([ars, ars]), np.concatenate([seg_u, seg_col]),
               np.concatenate([seg_w, -np.ones(ns)]), 0.0)

    # flow rows                                                          (:351-369)
    # Emitted straight in canonical CSR form: build_model's entries of a flow
    # row are (p', u) pairs per generator then the buses' slack columns; sorted
    # by column (SparseMatrix.from_coo) that is the u block (ascending unit),
    # the p' block, then the slack block, so each row is three slices and no
    # global sort over the (up to ~10^9) flow entries is needed.
    monitored = sorted(set(monitored))
    flow = None
    if monitored:
        if ptdf is None:
            needed = {}
            for lid, t, key in monitored:
                needed.setdefault(key, []).append(inst.line_pos[lid])
            ptdf = PtdfRows(inst.net, method=ptdf_method, device=device, needed=needed)
        gb = inst.gen_bus
        lens = np.empty(2 * len(monitored), np.int64)
        parts_c, parts_v, fr_rhs = [], [], np.empty(2 * len(monitored))
        for q, (lid, t, key) in enumerate(monitored):
            lpos = inst.line_pos[lid]
            delta = ptdf.row(lpos, key)
            limit = inst.limit[lpos] if key == BASE_CASE else inst.elimit[lpos]
            base = float(delta @ demand[:, t])
            coeff = delta[gb]
            gsel = np.flatnonzero(np.abs(coeff) > _FLOW_COEFF_DROP)
            bsel = np.flatnonzero(np.abs(delta) > _FLOW_COEFF_DROP)
            vu = coeff[gsel] * inst.pmin[gsel]
            ku = vu != 0.0                      # add_row drops exact zeros (:246)
            cols = np.concatenate([u[gsel[ku] * T + t], pp[gsel * T + t], pen[bsel * T + t]])
            vals = np.concatenate([vu[ku], coeff[gsel], delta[bsel]])
            parts_c.append(cols)
            parts_v.append(vals)
            lens[2 * q] = lens[2 * q + 1] = cols.size
            fr_rhs[2 * q], fr_rhs[2 * q + 1] = -limit + base, -limit - base
        flow = (lens, parts_c, parts_v, fr_rhs)

    # ---- bounds, objective -------------------------------------------------
    lower = np.zeros(n)
    upper = np.zeros(n)
    cost = np.zeros(n)
    upper[u] = 1.0
    upper[v] = 1.0
    upper[w] = 1.0
    on_win = np.where(inst.init_on == 1,
                      np.minimum(T, np.maximum(0, inst.min_up - inst.init_per)), 0)
    off_win = np.where(inst.init_on == 0,
                       np.minimum(T, np.maximum(0, inst.min_down - inst.init_per)), 0)
    lower[u[t_of < on_win[g_of]]] = 1.0
    upper[u[t_of < off_win[g_of]]] = 0.0
    upper[pp] = (inst.pmax - inst.pmin)[g_of]
    upper[seg_col] = seg_w
    cl = np.zeros(G)
    cu = np.zeros(G)
    for g in range(G):
        # builtin sum() (compensated since Python 3.12), exactly as :396-397
        pairs = list(zip(inst.seg_costs[g], inst.widths(g)))
        cl[g] = sum(min(0.0, c) * wd for c, wd in pairs)
        cu[g] = sum(max(0.0, c) * wd for c, wd in pairs)
    lower[cst] = cl[g_of]
    upper[cst] = cu[g_of]
    cost[cst] = 1.0
    cost[u] = inst.min_cost[g_of]
    upper[pen] = demand.reshape(-1)
    cost[pen] = inst.penalty

    # ---- canonical CSR (SparseMatrix.from_coo: sum dupes, drop zeros, sort) --
    r_all = np.concatenate(rows.r)
    c_all = np.concatenate(rows.c)
    v_all = np.concatenate(rows.v)
    m = rows.n
    order = np.argsort(r_all * np.int64(n) + c_all, kind="stable")
    r_all, c_all, v_all = r_all[order], c_all[order], v_all[order]
    dup = np.flatnonzero((r_all[1:] == r_all[:-1]) & (c_all[1:] == c_all[:-1]))
    if dup.size:
        raise AssertionError("duplicate (row, col) entries in SCUC builder")
    indptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(indptr, r_all + 1, 1)
    indptr = np.cumsum(indptr)
    rhs = np.concatenate(rows.rhs)
    indices, data = c_all.astype(np.int32), v_all
    if flow is not None:                 # the flow rows close the row order (:351-369)
        lens, parts_c, parts_v, fr_rhs = flow
        nf = int(lens.sum())
        if indptr[-1] + nf >= 2 ** 31:
            raise ValueError("nnz exceeds int32 indexing")
        fidx = np.empty(nf, np.int32)
        fval = np.empty(nf, np.float64)
        pos = 0
        for cols, vals in zip(parts_c, parts_v):
            k = cols.size
            fidx[pos:pos + k] = cols
            fval[pos:pos + k] = vals
            fidx[pos + k:pos + 2 * k] = cols
            np.negative(vals, out=fval[pos + k:pos + 2 * k])
            pos += 2 * k
        indptr = np.concatenate([indptr, indptr[-1] + np.cumsum(lens)])
        indices = np.concatenate([indices, fidx])
        data = np.concatenate([data, fval])
        rhs = np.concatenate([rhs, fr_rhs])
        m += lens.size
    if indptr[-1] >= 2 ** 31:
        raise ValueError("nnz exceeds int32 indexing")
    return LpArrays(indptr=indptr.astype(np.int32), indices=indices,
                    data=data, shape=(m, n), rhs=rhs,
                    cost=cost, lower=lower, upper=upper, n_eq=int(n_eq), offset=0.0)


def build_config(name: str, n_triples: int | None = None, ptdf_method: str | None = None,
                 device=None, seed: int | None = None):
    """Instance + LP for a named config.  C1 monitors all base triples by
    default; C2-C4 draw `n_triples` base triples.

    The PTDF rows are solved on the host under the pinned BLAS pool
    (``PTDF_BLAS_THREADS``) unless `device` is given explicitly, so the LP is
    bit-identical wherever it is built; tests/golden/*_trajectory.json and
    c4_window.json carry the digests the GPU parity tests assert."""
    with _blas_pool(BUILD_BLAS_THREADS):
        return _build_config(name, n_triples, ptdf_method, device, seed)


def _build_config(name, n_triples, ptdf_method, device, seed):
    cfg = dict(CONFIGS[name])
    if seed is not None:
        cfg["seed"] = seed
    doc = generate_instance(**cfg)
    if n_triples is None:
        n_triples = {"C1": -1, "C2": 500, "C3": 2000, "C4": 1000, "C5": 20000}[name]
    n1 = name == "C5"
    mon = all_base_triples(doc) if n_triples < 0 else sample_monitored(
        doc, n_triples, cfg["seed"], contingencies=n1)
    if ptdf_method is None:
        ptdf_method = ("lodf" if n1 else
                       "reference" if len(doc["buses"]) <= 2000 else "direct")
    if n1 and device is None:
        # ~20K base PTDF rows: one dense solve on the GPU when there is one
        # (C5 has no CPU reference run to reproduce, so no pinned host solve)
        try:
            import torch
            device = "cuda" if torch.cuda.is_available() else None
        except ImportError:
            device = None
    lp = build_relaxation(doc, mon, ptdf_method=ptdf_method, device=device)
    return doc, mon, lp
