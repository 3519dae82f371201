"""solve_many: independent LP solves overlapped on one
GPU give exactly the results of one-at-a-time solve() calls."""

import numpy as np
import pytest

from tests import golden_io

pytestmark = pytest.mark.gpu


def test_solve_many_matches_sequential():
    from paper_2510_10891_b200 import hprlp
    lps = [golden_io.random_lps()[i][0] for i in range(8)]
    cfg = hprlp.SolverConfig(tolerance=1e-6, log_residuals=True)
    seq = [hprlp.solve(lp, cfg) for lp in lps]
    par = hprlp.solve_many(lps, cfg, workers=8)
    for a, b in zip(seq, par):
        assert a.status == b.status and a.iterations == b.iterations
        assert a.restarts == b.restarts and a.lam == b.lam
        assert a.objective == b.objective
        assert a.x.tobytes() == b.x.tobytes() and a.y.tobytes() == b.y.tobytes()
        assert [r["rel_gap"] for r in a.residual_log] == [r["rel_gap"] for r in b.residual_log]


def test_solve_many_warm_starts_and_edges():
    from paper_2510_10891_b200 import hprlp
    lps = [golden_io.random_lps()[i][0] for i in (1, 2, 3)]
    cfg = hprlp.SolverConfig(tolerance=1e-6)
    first = hprlp.solve_many(lps, cfg)
    starts = [(r.x, r.y, r.z) for r in first]
    warm = hprlp.solve_many(lps, cfg, starts=starts, workers=2)
    for lp, w, s in zip(lps, warm, starts):
        ref = hprlp.solve(lp, cfg, start=s)
        assert w.iterations == ref.iterations and w.objective == ref.objective
    assert hprlp.solve_many([], cfg) == []
    with pytest.raises(ValueError):
        hprlp.solve_many(lps, cfg, starts=starts[:1])


def test_solve_many_duplicate_entries_get_private_engines():
    """The same LP object twice (and a second LP sharing its matrix and
    vectors, e.g. two warm starts of one node LP): every entry gets its own
    engine -- one handle is never driven by two threads -- and each result
    equals a lone solve (shared engine_for cache)."""
    import torch
    from paper_2510_10891_b200 import hprlp
    lp = golden_io.random_lps()[5][0]
    cfg = hprlp.SolverConfig(tolerance=1e-7)
    ref = hprlp.solve(lp, cfg)
    dev = torch.cuda.current_device()
    out = hprlp.solve_many([lp, lp, lp, lp], cfg, workers=4)
    assert torch.cuda.current_device() == dev
    for r in out:
        assert r.iterations == ref.iterations and r.objective == ref.objective
        assert r.x.tobytes() == ref.x.tobytes()
