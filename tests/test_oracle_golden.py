"""Pin the CPU oracle (oracle/hpr_oracle.py) against golden vectors that the
unmodified reference produced (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from oracle import hpr_oracle as O
from tests import golden_io
from tests.conftest import needs_reference


def _one_d():
    return golden_io.FixtureLp(np.array([0, 1]), np.array([0]), np.array([1.0]), (1, 1), [1.0],
                               [1.0], [0.0], [2.0], 0)


def test_kat_fixed_point_and_first_step():
    k = golden_io.kat()
    p = O.Problem.from_lp(_one_d())
    st = O.HprIterate([1.0], [1.0], [0.0], 1.0, 1.0, np.float64)
    st.step(p)
    assert [st.x[0], st.y[0], st.z[0]] == k["fixed_point_after"]
    r = O.kkt(p, [1.0], [1.0], [0.0])
    assert [r.primal, r.box, r.dual] == k["fixed_point_kkt"] == [0.0, 0.0, 0.0]
    st = O.HprIterate([0.0], [0.0], [0.0], 1.0, 1.0, np.float64)
    st.step(p)
    assert [st.bx[0], st.by[0], st.bz[0]] == k["from_zero_bar"] == [0.0, 1.0, 1.0]
    assert [st.x[0], st.y[0], st.z[0]] == k["from_zero_next"]
    assert O.kkt(p, [0.5], [0.0], [0.0]).primal == k["primal_residual_x05"] == 0.5


def test_kat_power_method():
    import scipy.sparse as sp
    k = golden_io.kat()
    eye = O.Csr(sp.eye(3, format="csr"))
    assert O.power_lambda(eye, 1e-4, 1000, 0, None) == k["power_identity"]
    assert O.power_lambda(eye, 1e-4, 1000, 0, 1.01) == k["power_identity_solve_inflation"]
    d = O.Csr(sp.diags([2.0, 1.0], format="csr"))
    assert O.power_lambda(d, 1e-4, 1000, 0, None) == k["power_diag21"]


def test_kat_one_d_solve():
    k = golden_io.kat()["one_d_solve"]
    r = O.solve(_one_d(), O.OracleConfig(tolerance=1e-8))
    assert r.status == k["status"] and r.iterations == k["iterations"]
    assert r.objective == k["objective"] and r.x.tolist() == k["x"]


CFGS = {"fp64": dict(tolerance=1e-8), "fp32": dict(tolerance=1e-6, precision="fp32"),
        "fp64_noruiz_log": dict(tolerance=1e-6, ruiz=False, log_residuals=True)}


@pytest.mark.parametrize("tag", list(CFGS))
def test_random_lps_bit_identical(tag):
    for lp, rec, res in golden_io.random_lps():
        r = O.solve(lp, O.OracleConfig(**CFGS[tag]))
        g = res[tag]
        assert r.status == g["status"]
        assert (r.iterations, r.restarts) == (g["iterations"], g["restarts"])
        assert r.lam == g["lam"] and r.sigma_final == g["sigma_final"]
        assert r.objective == g["objective"]
        assert np.array_equal(r.x, g["x"]) and np.array_equal(r.y, g["y"])
        assert np.array_equal(r.z, g["z"])
        if "log" in g:
            mine = np.array([[e["iteration"], e["epoch"], e["rel_primal"], e["rel_dual"],
                              e["rel_box"], e["rel_gap"], e["sigma"]] for e in r.residual_log])
            assert np.array_equal(mine, g["log"])


def test_random_lps_match_highs():
    for lp, rec, res in golden_io.random_lps():
        obj, hi = res["fp64"]["objective"], rec["highs_objective"]
        assert abs(obj - hi) <= 1e-6 * max(1.0, abs(hi))


@pytest.mark.parametrize("tag,cfg", [
    ("fp64_1e4", dict(tolerance=1e-4, ruiz=False, log_residuals=True)),
    ("fp64_1e6_ruiz", dict(tolerance=1e-6, ruiz=True, log_residuals=True, max_iterations=20000)),
])
def test_scuc_small_trajectory(tag, cfg):
    lp, meta, res = golden_io.scuc_small()
    r = O.solve(lp, O.OracleConfig(**cfg))
    g = res[tag]
    assert r.status == g["status"] and r.iterations == g["iterations"]
    assert r.restarts == g["restarts"] and r.objective == g["objective"]
    mine = np.array([[e["iteration"], e["epoch"], e["rel_primal"], e["rel_dual"], e["rel_box"],
                      e["rel_gap"], e["sigma"]] for e in r.residual_log])
    assert np.array_equal(mine, g["log"])


@needs_reference
def test_oracle_equals_reference_directly():
    """Cross-check on fresh random LPs against the live reference."""
    from scuckit import hprlp, lp_kernel
    from tests.golden.make_golden import random_lp
    rng = np.random.default_rng(99)
    for _ in range(5):
        d = random_lp(rng)
        lp = golden_io.FixtureLp(**d)
        ref_lp = lp_kernel.StandardFormLp(matrix=lp_kernel.SparseMatrix(lp.matrix.csr),
                                          rhs=lp.rhs, cost=lp.cost, lower=lp.lower,
                                          upper=lp.upper, n_eq=lp.n_eq)
        a = hprlp.solve(ref_lp, hprlp.SolverConfig(tolerance=1e-7, log_residuals=True))
        b = O.solve(lp, O.OracleConfig(tolerance=1e-7, log_residuals=True))
        assert a.iterations == b.iterations and a.objective == b.objective
        assert np.array_equal(a.x, b.x) and a.residual_log == b.residual_log


def test_oracle_config_variants_match_reference():
    """Every SolverConfig field the driver leaves at its default, moved
    (tests/golden/config_variants.json, unmodified reference): the oracle
    reproduces status, iterations, restarts, lambda, sigma and the objective."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config_variants.json")))
    lps = golden_io.random_lps()[:8]
    for key, rec in g["results"].items():
        i, name = key.split("/")
        r = O.solve(lps[int(i)][0], O.OracleConfig(**g["variants"][name]))
        assert r.status == rec["status"], key
        assert r.iterations == rec["iterations"] and r.restarts == rec["restarts"], key
        assert r.lam == rec["lam"], key
        assert r.sigma_final == rec["sigma_final"], key
        assert r.objective == rec["objective"], key


def test_oracle_warm_starts_match_reference():
    """Solves started from a perturbed optimum (B&B's start=), FP64 and FP32,
    against the reference's records (tests/golden/warm_starts.npz)."""
    from paper_2510_10891_b200.lp import Precision  # noqa: F401
    lps = golden_io.random_lps()[:6]
    for (lp, _, _), (start, rec) in zip(lps, golden_io.warm_starts()):
        for prec, tol in (("fp64", 1e-7), ("fp32", 1e-5)):
            r = O.solve(lp, O.OracleConfig(tolerance=tol, precision=prec), start=start)
            g = rec[prec]
            assert r.status == g["status"]
            assert (r.iterations, r.restarts) == (g["iterations"], g["restarts"])
            assert r.objective == g["objective"] and r.lam == g["lam"]
