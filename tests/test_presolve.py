"""Native presolve core (include/hpr_presolve.h) vs the reference presolve
(scuckit/presolve.py): identical reduced models, reduction logs and
infeasibility certificates.  CPU only — the core never touches the GPU."""

import json
import os
import sys
import types

import numpy as np
import pytest

from paper_2510_10891_b200 import lp as L
from paper_2510_10891_b200 import presolve as P
from tests.presolve_cases import digest, random_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MIRROR = types.SimpleNamespace(SparseMatrix=L.SparseMatrix, StandardFormLp=L.StandardFormLp,
                               MilpModel=L.MilpModel)


def _reference():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "scuckit")) and p not in sys.path:
            sys.path.append(p)
    try:
        import scuckit.presolve  # noqa: F401
        return True
    except Exception:
        return False


needs_reference = pytest.mark.skipif(not _reference(), reason="reference package not importable")


def test_golden_digests():
    """60 seeded MILPs: every rule and every certificate kind, against the
    reference's own outputs (tests/golden/presolve.json)."""
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "presolve.json")))
    kinds = set()
    for seed, rec in g.items():
        model, _ = random_case(int(seed), MIRROR)
        red, log = P.milp_presolve(model)
        assert log.infeasible == rec["infeasible"], seed
        assert digest((red, log)) == rec["milp"], seed
        if "lp" in rec:
            res = P.lp_presolve(red.relax())
            assert res[1].infeasible == rec["lp_infeasible"]
            assert digest(res) == rec["lp"], seed
        kinds.add((rec["infeasible"] or "feasible").split(" ")[0])
    assert kinds == {"feasible", "row", "column"}


def _same(a, b):
    (ma, la), (mb, lb) = a, b
    for k in ("kept_cols", "kept_rows"):
        assert np.array_equal(getattr(la, k), getattr(lb, k)), k
    for k in ("fixed_values", "removed_rows", "bound_changes", "objective_delta", "infeasible"):
        assert getattr(la, k) == getattr(lb, k), k
    pa = ma.lp if hasattr(ma, "lp") else ma
    pb = mb.lp if hasattr(mb, "lp") else mb
    ca, cb = pa.matrix.csr, pb.matrix.csr
    assert np.array_equal(ca.indptr, cb.indptr) and np.array_equal(ca.indices, cb.indices)
    assert np.array_equal(ca.data, cb.data)
    assert (ca.indptr.dtype, ca.indices.dtype, ca.data.dtype) == (cb.indptr.dtype,
                                                                  cb.indices.dtype, cb.data.dtype)
    for k in ("rhs", "cost", "lower", "upper"):
        assert np.array_equal(getattr(pa, k), getattr(pb, k)), k
    assert (pa.n_eq, pa.offset, pa.row_tags, pa.col_tags) == (pb.n_eq, pb.offset, pb.row_tags,
                                                              pb.col_tags)


@needs_reference
def test_c1_bit_identical_to_reference():
    """C1 (118 buses, 54 units, 24 periods, all base flow rows): milp_presolve,
    lp_presolve of its relaxation, and milp_presolve after the reference's own
    round-1 fixes (tests/golden/c1_fixing.json), whose certificate is the one
    the reference's fixing loop raises."""
    from scuckit import apply_instance_scaling, build_model, parse_instance
    from scuckit import presolve as R
    from paper_2510_10891_b200 import scuc
    doc = scuc.generate_instance(**scuc.CONFIGS["C1"])
    inst, _ = apply_instance_scaling(parse_instance(doc))
    model, _ = build_model(inst, monitored=scuc.all_base_triples(doc))
    P._LOG_CLASS = R.ReductionLog
    try:
        ref = R.milp_presolve(model)
        _same(ref, P.milp_presolve(model))
        assert len(ref[1].bound_changes) > 100 and len(ref[1].removed_rows) > 1000
        lp = ref[0].relax()
        _same(R.lp_presolve(lp), P.lp_presolve(lp))
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "c1_fixing.json")))
        for k, v in g["fixed"].items():
            model.fix_column(int(k), float(v), "golden round 1")
        ref = R.milp_presolve(model)
        _same(ref, P.milp_presolve(model))
        assert ref[1].infeasible and ref[1].infeasible in g["error"]
    finally:
        P._LOG_CLASS = P.ReductionLog


@needs_reference
def test_install_rebinds_presolve_everywhere():
    import scuckit
    import scuckit.fixing
    import scuckit.milp_bb
    import scuckit.presolve
    from paper_2510_10891_b200 import hprlp
    orig = scuckit.fixing.milp_presolve
    hprlp.install()
    try:
        for mod in (scuckit, scuckit.fixing, scuckit.milp_bb, scuckit.presolve):
            assert mod.milp_presolve is P.milp_presolve and mod.lp_presolve is P.lp_presolve
        assert P._LOG_CLASS is scuckit.presolve.ReductionLog
    finally:
        hprlp.uninstall()
    assert scuckit.fixing.milp_presolve is orig and P._LOG_CLASS is P.ReductionLog


def test_uncrush_and_log_mirror():
    log = P.ReductionLog(n_cols_full=5, n_rows_full=2,
                         kept_cols=np.array([0, 2, 4]), fixed_values={1: 3.0, 3: -1.0})
    assert np.array_equal(P.uncrush(np.array([1.0, 2.0, 5.0]), log), [1, 3, 2, -1, 5])
    with pytest.raises(ValueError):
        P.uncrush(np.zeros(4), log)
    assert log.feasible


def test_native_rejects_bad_input():
    import ctypes as C
    from paper_2510_10891_b200 import _capi
    lib = _capi.load()
    h = C.c_void_p()
    assert lib.hpr_presolve_run(None, 100, C.byref(h)) != 0


def test_native_submatrix_matches_scipy_fancy_indexing():
    """hpr_presolve_reduce returns exactly csr[rows][:, cols] (presolve.py:244,
    :278): same arrays, same dtypes, including empty selections, empty rows
    and a matrix whose column row-lists the core builds itself."""
    import scipy.sparse as sp
    rng = np.random.default_rng(7)
    for trial in range(12):
        m, n = int(rng.integers(0, 60)), int(rng.integers(1, 50))
        a = sp.random(m, n, density=float(rng.uniform(0.0, 0.4)), random_state=trial,
                      format="csr")
        a.data[rng.random(a.nnz) < 0.1] = -1.5               # some repeated values
        lp = L.StandardFormLp(matrix=L.SparseMatrix(a), rhs=np.zeros(m), cost=np.zeros(n),
                              lower=np.zeros(n), upper=np.ones(n), n_eq=0)
        red = P._Reduction(lp, None)
        rows = rng.random(m) < rng.uniform(0.0, 1.0)
        cols = rng.random(n) < rng.uniform(0.0, 1.0)
        if trial == 0:
            rows[:] = False
        if trial == 1:
            cols[:] = False
        ref = red.csr[np.flatnonzero(rows)][:, np.flatnonzero(cols)]
        got = red.submatrix(rows, cols)
        assert got.shape == ref.shape
        for k in ("indptr", "indices", "data"):
            x, y = getattr(got, k), getattr(ref, k)
            assert x.dtype == y.dtype and np.array_equal(x, y), (trial, k)
        ref = red.csr[np.flatnonzero(rows)]
        got = red.submatrix(rows)
        for k in ("indptr", "indices", "data"):
            x, y = getattr(got, k), getattr(ref, k)
            assert x.dtype == y.dtype and np.array_equal(x, y), (trial, k)
