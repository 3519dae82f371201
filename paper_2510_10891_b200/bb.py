"""Speculative sibling solves for the reference's branch-and-bound
(B&B node LPs batched in the real flow).

The reference searches best-first with depth-first plunging until the first
incumbent exists (``milp_bb.py:279-404``): at a branching node the preferred
child is evaluated at once and its sibling goes onto the heap, to be popped
when the dive ends.  Each evaluation is one small warm-started node LP at
tolerance 1e-6 (``_evaluate``, ``milp_bb.py:204-253``) -- a size the GPU
engine runs far below its capacity.

``SpeculativeSearch`` is the reference's ``_Search`` with one addition: when
a plunge pushes a sibling, that sibling's node LP is prepared and solved
ahead, on a worker thread with its own engine and CUDA stream, while the
dive goes on.  When the search later evaluates the sibling, the reference's
own ``_evaluate`` runs unchanged; its ``lp_backends.solve_lp`` call is
answered from the speculative result if -- and only if -- the LP, the warm
start and the solver configuration are identical (the time limit aside) and
the speculative solve did not stop on its time limit.  The engine is
deterministic and a solve on a private engine is bit-identical to a lone
solve (``tests/test_gpu_batch.py``), so every node result, hence the search
order, the incumbents and the final MILP result, is the reference's.  A
sibling that is pruned before it is popped costs only GPU time that would
otherwise idle.

``hprlp.install()`` rebinds ``scuckit.milp_bb._Search`` to it (module
lookup in ``solve_milp``, ``milp_bb.py:407-412``) and wraps
``scuckit.lp_backends.solve_lp``; outside a speculative evaluation the
wrapper is a pass-through.
"""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_CTX = threading.local()
STATS = {"speculated": 0, "hits": 0, "misses": 0}


def _same_lp(a, b) -> bool:
    if a is b:
        return True
    ca, cb = a.matrix.csr, b.matrix.csr
    if ca.shape != cb.shape or a.n_eq != b.n_eq or float(a.offset) != float(b.offset):
        return False
    return (np.array_equal(ca.indptr, cb.indptr) and np.array_equal(ca.indices, cb.indices)
            and np.array_equal(ca.data, cb.data)
            and all(np.array_equal(getattr(a, f), getattr(b, f))
                    for f in ("rhs", "cost", "lower", "upper")))


def _same_start(a, b) -> bool:
    if a is None or b is None:
        return a is None and b is None
    return all(np.array_equal(np.asarray(u), np.asarray(v)) for u, v in zip(a, b))


def _cfg_key(cfg) -> dict:
    d = dict(cfg.__dict__)
    d.pop("time_limit", None)
    return d


def wrap_solve_lp(orig):
    """``lp_backends.solve_lp`` answering a speculative evaluation's node LP
    from the prepared result when it is provably the same solve."""
    def solve_lp(lp, backend="hpr", config=None, start=None):
        ent = getattr(_CTX, "entry", None)
        if ent is not None and backend == "hpr" and config is not None:
            _CTX.entry = None                        # one LP per evaluation
            got = ent()                              # waits for the speculative solve
            if got is not None:
                lp2, warm, cfg, sol = got
                if (_cfg_key(cfg) == _cfg_key(config) and sol.status != "time-limit"
                        and (config.time_limit is None or sol.solve_time < config.time_limit)
                        and _same_lp(lp2, lp) and _same_start(warm, start)):
                    STATS["hits"] += 1
                    return sol
            STATS["misses"] += 1
        return orig(lp, backend=backend, config=config, start=start)
    solve_lp.__wrapped__ = orig
    return solve_lp


def make_search_class(milp_bb, lp_backends):
    """The reference's ``_Search`` (this module's docstring) as a subclass."""
    base = milp_bb._Search
    if getattr(base, "_speculative", False):
        return base

    class SpeculativeSearch(base):
        _speculative = True

        def __init__(self, *args, **kw):
            super().__init__(*args, **kw)
            self._spec = {}
            self._stream = None
            self._pool = ThreadPoolExecutor(max_workers=1)
            import torch
            self._device = torch.cuda.current_device() if torch.cuda.is_available() else None

        def _prepare(self, node):
            """The LP ``_evaluate`` would solve for `node` (milp_bb.py:204-236),
            or None when it would not reach a solve."""
            nodem = self.base.copy()
            for col, val in node.fixes:
                nodem.lp.lower[col] = val
                nodem.lp.upper[col] = val
            reduced, mlog = milp_bb.milp_presolve(nodem)
            if not mlog.feasible:
                return None
            lp2, llog = milp_bb.lp_presolve(reduced.relax())
            if not llog.feasible or lp2.n_rows == 0:
                return None
            return lp2, self._warm_restrict(node.warm, mlog, llog)

        def _solve_ahead(self, node, cfg):
            import torch
            from . import hprlp
            if self._device is not None:
                torch.cuda.set_device(self._device)
            prep = self._prepare(node)
            if prep is None:
                return None, None
            lp2, warm = prep
            # a default-priority stream: the search's own solves run on the
            # engine's greatest-priority private streams, so the speculative
            # work only takes SMs they leave idle
            if self._stream is None:
                self._stream = torch.cuda.Stream(device=self._device, priority=0)
            eng = hprlp.Engine(lp2, device=self._device, stream=self._stream)
            try:
                res = hprlp._with_fp64_retry(
                    cfg, lambda c, t0: hprlp._solve_once(lp2, c, warm, t0, engine=eng))
            finally:
                eng.close()
            sol = lp_backends.LpSolution(
                x=res.x, y=res.y, z=res.z, objective=res.objective,
                status=res.status.value, converged=res.converged, solve_time=res.solve_time,
                iterations=res.iterations, residual_log=res.residual_log or None)
            return (lp2, warm), sol

        def _speculate(self, node):
            if node.bound >= self._cutoff():
                return
            left = self._time_left()
            if left is not None and left <= 0.0:
                return
            cfg = self.lp_cfg
            if left is not None:                     # as _evaluate (milp_bb.py:233-236)
                cfg = type(cfg)(**{**cfg.__dict__,
                                   "time_limit": max(0.1, left) if cfg.time_limit is None
                                   else min(cfg.time_limit, max(0.1, left))})
            self._spec[node.seq] = (cfg, self._pool.submit(self._solve_ahead, node, cfg))
            STATS["speculated"] += 1

        def _pending(self) -> int:
            return sum(1 for _, f in self._spec.values() if not f.done())

        def _process(self, node, is_root):
            if node.bound >= self._cutoff():         # pruned without evaluation
                ent = self._spec.pop(node.seq, None)
                if ent is not None:
                    ent[1].cancel()
            seq0 = self.seq
            plunge_child = super()._process(node, is_root)
            if plunge_child is not None:
                # a plunge: the child is evaluated next, its sibling waits on the heap
                for n in self.heap:
                    if n.seq >= seq0 and n.seq != plunge_child.seq:
                        self._speculate(n)
            elif len(self.heap) > 1 and self._pending() < 2:
                # best-first: heap[0] is popped next; the runner-up is likely after it
                # (children of heap[0] inherit its bound, which is no smaller)
                nxt = min(self.heap[1:3])
                if nxt.seq not in self._spec and nxt.bound < self._cutoff():
                    self._speculate(nxt)
            return plunge_child

        def _evaluate(self, node):
            ent = self._spec.pop(node.seq, None)
            if ent is not None:
                cfg, fut = ent

                def entry():
                    if fut.cancel():                 # still queued: solve it directly
                        return None
                    try:
                        prep, sol = fut.result()
                    except Exception:                # the direct solve reports any error
                        return None
                    return None if prep is None else (prep[0], prep[1], cfg, sol)
                _CTX.entry = entry
            try:
                return super()._evaluate(node)
            finally:
                _CTX.entry = None

        def run(self, initial_incumbent):
            try:
                return super().run(initial_incumbent)
            finally:
                for cfg, fut in self._spec.values():
                    fut.cancel()
                self._pool.shutdown(wait=True)

    SpeculativeSearch.__name__ = base.__name__
    SpeculativeSearch.__qualname__ = base.__qualname__
    return SpeculativeSearch
