"""The vectorised SCUC LP builder reproduces the reference build_model."""

import numpy as np
import pytest

from paper_2510_10891_b200 import scuc
from tests.conftest import needs_reference


def sizes(doc, n_mon):
    G, B, T = len(doc["generators"]), len(doc["buses"]), doc["time_periods"]
    H = sum(len(g["segments"]) for g in doc["generators"])
    return dict(n=5 * G * T + T * H + B * T, n_eq=3 * G * T + T,
                m=9 * G * T + T + T * H + 2 * n_mon)


@pytest.mark.parametrize("args", [(6, 5, 8, 6, 0), (30, 12, 45, 8, 3), (60, 20, 90, 12, 7)])
def test_size_formulas(args):
    B, G, L, T, seed = args
    doc = scuc.generate_instance(B, G, L, T, seed=seed)
    mon = scuc.sample_monitored(doc, 10, seed)
    lp = scuc.build_relaxation(doc, mon)
    s = sizes(doc, len(set(mon)))
    assert lp.shape == (s["m"], s["n"]) and lp.n_eq == s["n_eq"]
    # flow row pairs are exact negatives (formulation.py:366-369)
    csr = lp.csr()
    lo = csr[lp.shape[0] - 2].toarray()
    hi = csr[lp.shape[0] - 1].toarray()
    assert np.array_equal(lo, -hi)


def test_generator_is_deterministic():
    a = scuc.generate_instance(30, 12, 45, 8, seed=3)
    b = scuc.generate_instance(30, 12, 45, 8, seed=3)
    assert a == b
    la = scuc.build_relaxation(a, scuc.all_base_triples(a))
    lb = scuc.build_relaxation(b, scuc.all_base_triples(b))
    assert la.digest() == lb.digest()


@needs_reference
@pytest.mark.parametrize("args", [(6, 5, 8, 6, 0, -1), (30, 12, 45, 8, 3, -1),
                                  (60, 20, 90, 12, 7, 40), (118, 54, 186, 24, 1, 300)])
def test_csr_identical_to_reference_build_model(args):
    from scuckit import build_model, parse_instance
    B, G, L, T, seed, ntr = args
    doc = scuc.generate_instance(B, G, L, T, seed=seed)
    mon = scuc.all_base_triples(doc) if ntr < 0 else scuc.sample_monitored(doc, ntr, seed)
    mine = scuc.build_relaxation(doc, mon)
    ref = build_model(parse_instance(doc), monitored=mon)[0].relax()
    c = ref.matrix.csr
    assert c.shape == mine.shape and ref.n_eq == mine.n_eq
    assert np.array_equal(c.indptr, mine.indptr) and np.array_equal(c.indices, mine.indices)
    assert np.array_equal(c.data, mine.data)
    for a, b in ((ref.rhs, mine.rhs), (ref.cost, mine.cost), (ref.lower, mine.lower),
                 (ref.upper, mine.upper)):
        assert np.array_equal(a, b)


@needs_reference
def test_direct_ptdf_rows_match_reference_tables():
    from scuckit import compute_ptdf, parse_instance
    doc = scuc.generate_instance(60, 20, 90, 12, seed=7, n_contingencies=3)
    inst = scuc.Instance(doc)
    ref = compute_ptdf(parse_instance(doc).network)
    lines = [0, 5, 70, 89]
    for key in ["base"] + [c["id"] for c in doc["contingencies"]]:
        skip = None if key == "base" else inst.net.cont_line[key]
        rows = scuc._ptdf_rows_direct(inst.B, inst.net.fb, inst.net.tb, inst.net.react,
                                      inst.net.ref, lines, skip=skip)
        np.testing.assert_allclose(rows, ref.table(key)[lines], rtol=0, atol=1e-12)


def test_c1_digest_matches_golden_fixture():
    """The C1 LP this builder makes is the one the reference trajectory
    fixture (tests/golden/c1_trajectory.json) was recorded on."""
    from tests import golden_io
    g = golden_io.c1()
    doc, mon, lp = scuc.build_config("C1")
    assert lp.shape == tuple(g["shape"]) and lp.nnz == g["nnz"]
    assert lp.digest() == g["digest"]


@needs_reference
def test_lodf_rows_match_refactorised_contingency_tables():
    """C5's contingency rows: the LODF update from the base rows equals the
    reference's per-contingency refactorisation (compute_ptdf,
    instance.py:241-267) to rounding, including the zeroed outaged row."""
    from scuckit import compute_ptdf, parse_instance
    doc = scuc.generate_instance(60, 20, 90, 12, seed=7, n_contingencies=5)
    inst = scuc.Instance(doc)
    ref = compute_ptdf(parse_instance(doc).network)
    keys = [c["id"] for c in doc["contingencies"]]
    lines = list(range(len(doc["lines"])))
    needed = {k: lines for k in keys}
    prov = scuc.PtdfRows(inst.net, method="lodf", needed=needed)
    for key in keys:
        got = np.stack([prov.row(q, key) for q in lines])
        want = ref.table(key)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)
        k = inst.net.cont_line[key]
        assert not got[k].any() and not got[:, inst.net.ref].any()


@needs_reference
@pytest.mark.parametrize("ptdf_method", ["reference", "lodf"])
def test_n1_flow_rows_match_reference_build_model(ptdf_method):
    """N-1 monitored triples (the C5 row family): CSR structure, rhs and
    values against build_model on the reference's own contingency tables --
    identical with the refactorised tables, within rounding with the LODF
    rows (the reference's 1e-10 coefficient drop decides the same way)."""
    from scuckit import build_model, compute_ptdf, parse_instance
    doc = scuc.generate_instance(60, 20, 90, 12, seed=7, n_contingencies=4)
    mon = scuc.sample_monitored(doc, 120, 7, contingencies=True)
    mine = scuc.build_relaxation(doc, mon, ptdf_method=ptdf_method)
    inst = parse_instance(doc)
    ref = build_model(inst, monitored=mon, ptdf=compute_ptdf(inst.network))[0].relax()
    c = ref.matrix.csr
    assert c.shape == mine.shape
    assert np.array_equal(c.indptr, mine.indptr) and np.array_equal(c.indices, mine.indices)
    if ptdf_method == "reference":
        assert np.array_equal(c.data, mine.data) and np.array_equal(ref.rhs, mine.rhs)
    else:
        np.testing.assert_allclose(mine.data, c.data, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(mine.rhs, ref.rhs, rtol=1e-10, atol=1e-9)


def _same_model(a, b):
    la, lb = a[0].lp, b[0].lp
    ca, cb = la.matrix.csr, lb.matrix.csr
    assert ca.shape == cb.shape and la.n_eq == lb.n_eq
    assert np.array_equal(ca.indptr, cb.indptr) and np.array_equal(ca.indices, cb.indices)
    assert np.array_equal(ca.data, cb.data)
    for f in ("rhs", "cost", "lower", "upper"):
        assert np.array_equal(getattr(la, f), getattr(lb, f)), f
    assert la.row_tags == lb.row_tags and la.col_tags == lb.col_tags
    assert np.array_equal(a[0].integrality, b[0].integrality)
    assert a[1].n_cols == b[1].n_cols and np.array_equal(a[1].pprime, b[1].pprime)


@needs_reference
@pytest.mark.parametrize("args", [(30, 12, 45, 8, 3, -1, 0), (60, 20, 90, 12, 7, 40, 0),
                                  (118, 54, 186, 24, 1, 300, 0), (60, 20, 90, 12, 7, 80, 3)])
def test_dropin_build_model_identical_to_reference(args):
    """builder.build_model (the install()ed replacement) against the
    reference's build_model on the instance-scaled instance the driver uses
    (driver.py:211-212, :249-250): CSR, rhs, bounds, costs, row and column
    tags, integrality -- identical, with base and N-1 triples."""
    from scuckit import apply_instance_scaling, build_model, compute_ptdf, parse_instance
    from paper_2510_10891_b200 import builder
    B, G, L, T, seed, ntr, nc = args
    doc = scuc.generate_instance(B, G, L, T, seed=seed, n_contingencies=nc)
    inst = parse_instance(doc)
    ptdf = compute_ptdf(inst.network)
    work, _ = apply_instance_scaling(inst)
    mon = (scuc.all_base_triples(doc) if ntr < 0 else
           scuc.sample_monitored(doc, ntr, seed, contingencies=nc > 0))
    _same_model(builder.build_model(work, mon, ptdf), build_model(work, monitored=mon, ptdf=ptdf))
    _same_model(builder.build_model(work, (), ptdf), build_model(work, monitored=(), ptdf=ptdf))


@needs_reference
def test_dropin_build_model_errors_like_reference():
    from scuckit import build_model, parse_instance
    from scuckit.formulation import ModelError
    from paper_2510_10891_b200 import builder
    doc = scuc.generate_instance(12, 6, 18, 6, seed=5)
    inst = parse_instance(doc)
    for bad in [("l999", 0, "base"), ("l0", 6, "base"), ("l0", 0, "c9")]:
        with pytest.raises(ModelError) as mine:
            builder.build_model(inst, [bad])
        with pytest.raises(ModelError) as ref:
            build_model(inst, monitored=[bad])
        assert str(mine.value) == str(ref.value)


@needs_reference
def test_dropin_compute_ptdf_matches_reference():
    from scuckit import compute_ptdf, parse_instance
    from paper_2510_10891_b200 import builder
    doc = scuc.generate_instance(60, 20, 90, 12, seed=7, n_contingencies=4)
    net = parse_instance(doc).network
    a, b = builder.compute_ptdf(net, device=None), compute_ptdf(net)
    assert type(a) is type(b) and a.keys() == b.keys()
    assert a.line_ids == b.line_ids and a.bus_ids == b.bus_ids
    for k in b.keys():
        np.testing.assert_allclose(a.table(k), b.table(k), rtol=0, atol=1e-12)


@needs_reference
def test_install_rebinds_builder_everywhere():
    """install() routes the driver's per-pass model construction to the
    vectorised builder (driver.py:210, :249-250) and uninstall() restores it."""
    import scuckit
    import scuckit.driver
    import scuckit.formulation
    import scuckit.instance
    from paper_2510_10891_b200 import builder, hprlp
    orig = scuckit.driver.build_model, scuckit.driver.compute_ptdf
    hprlp.install()
    try:
        for mod in (scuckit, scuckit.driver, scuckit.formulation):
            assert mod.build_model is builder.build_model
        for mod in (scuckit, scuckit.driver, scuckit.formulation, scuckit.instance):
            assert mod.compute_ptdf is builder.compute_ptdf
    finally:
        hprlp.uninstall()
    assert (scuckit.driver.build_model, scuckit.driver.compute_ptdf) == orig
    assert scuckit.formulation.build_model is not builder.build_model
