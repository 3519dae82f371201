"""Flow screen: scuckit.driver.screen_violations
(driver.py:165-200) on the GPU.

CPU: oracle/screen_oracle.py reproduces the reference's violation lists in
tests/golden/screen.npz (made by tests/golden/make_screen_golden.py from the
unmodified reference) exactly, and the product's injection rebuild is
bit-identical to the oracle's.  GPU: the device screen returns the same
violations (same triples, order, limits and monitored flags; flows and
excesses within FP64 reassociation, 1e-12 of the row's |PTDF|.|inj| scale)
through the same Python signature, plus the contract's error behaviour."""

import json
import os

import numpy as np
import pytest

from oracle import screen_oracle
from paper_2510_10891_b200 import screen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "screen.npz")
N_CASES, N_POINTS = 4, 3


def golden():
    return np.load(GOLD)


_Line = screen._Line
instance_of = screen.instance_view


def _Ptdf(keys, tables):
    return screen.Tables(dict(zip(keys, tables)))


def case(g, ci):
    doc = json.loads(str(g[f"c{ci}_doc"]))
    inst = instance_of(doc)
    return doc, inst, _Ptdf(inst.contingency_keys(), g[f"c{ci}_tables"]), float(g[f"c{ci}_tol"])


def oracle_inj(doc, inst, x):
    bidx = inst.network.bus_index()
    return screen_oracle.injections(
        x, len(inst.generators), inst.n_periods, len(inst.buses),
        sum(g.n_segments for g in inst.generators), [g.p_min for g in inst.generators],
        [bidx[g.bus] for g in inst.generators], inst.demand_matrix())


def points(g, ci):
    for p in range(N_POINTS):
        mon = {tuple(m) for m in json.loads(str(g[f"c{ci}_p{p}_monitored"]))}
        yield g[f"c{ci}_p{p}_x"], mon, json.loads(str(g[f"c{ci}_p{p}_viol"]))


@pytest.mark.parametrize("ci", range(N_CASES))
def test_oracle_matches_reference_golden(ci):
    g = golden()
    doc, inst, ptdf, tol = case(g, ci)
    keys = inst.contingency_keys()
    for x, mon, ref in points(g, ci):
        inj = oracle_inj(doc, inst, x)
        got = screen_oracle.screen(g[f"c{ci}_tables"], g[f"c{ci}_limits"], keys,
                                   [ln.lid for ln in inst.lines], inj, mon, tol)
        assert [list(v) for v in got] == ref


@pytest.mark.parametrize("ci", range(N_CASES))
def test_injection_rebuild_is_bit_identical(ci):
    g = golden()
    doc, inst, _, _ = case(g, ci)
    for x, _, _ in points(g, ci):
        a = screen.injections(x, inst)
        b = oracle_inj(doc, inst, x)
        assert a.tobytes() == b.tobytes()


def test_point_length_is_checked():
    g = golden()
    _, inst, ptdf, _ = case(g, 0)
    with pytest.raises(ValueError, match="point length"):
        screen.screen_violations(np.zeros(7), inst, ptdf)


def _compare(got, ref, tables, inj):
    """Same violation set with the reference's limits and monitored flags,
    flows/excesses within FP64 reassociation (1e-12 of the |PTDF|.|inj|
    bound), in the reference's sort order: our list is exactly sorted by its
    own key, and position by position the excesses agree to the same bound
    (entries whose excesses tie to rounding may swap places)."""
    tol = 1e-12 * max(1.0, float((np.abs(tables) @ np.abs(inj)).max()))
    assert len(got) == len(ref)
    by = {(r[0], r[1], r[2]): r for r in ref}
    assert {v.triple for v in got} == set(by)
    for v in got:
        r = by[v.triple]
        assert v.limit == r[4] and v.already_monitored == r[6]
        assert abs(v.flow - r[3]) <= tol and abs(v.excess - r[5]) <= tol
    keys = [(-v.excess, v.line, v.period, v.contingency) for v in got]
    assert keys == sorted(keys)
    for v, r in zip(got, ref):
        assert abs(v.excess - r[5]) <= tol
        if (v.line, v.period, v.contingency) != (r[0], r[1], r[2]):
            assert abs(by[v.triple][5] - r[5]) <= 2 * tol   # a rounding tie


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(N_CASES))
def test_device_screen_matches_reference(ci):
    g = golden()
    doc, inst, ptdf, tol = case(g, ci)
    tabs = g[f"c{ci}_tables"]
    for x, mon, ref in points(g, ci):
        got = screen.screen_violations(x, inst, ptdf, monitored=mon, tol=tol)
        _compare(got, ref, tabs, screen.injections(x, inst))


@pytest.mark.gpu
def test_device_flows_and_resident_tables():
    g = golden()
    doc, inst, ptdf, tol = case(g, 3)
    x = g["c3_p0_x"]
    inj = screen.injections(x, inst)
    scr = screen.screen_for(ptdf, inst)
    assert screen.screen_for(ptdf, inst) is scr       # tables stay resident
    scr.run(inj, tol)
    for k in range(len(inst.contingency_keys())):
        want = g["c3_tables"][k] @ inj
        np.testing.assert_allclose(scr.flows(k), want, rtol=0,
                                   atol=1e-12 * max(1.0, np.abs(want).max()))
    info = scr.info()
    assert info["n_tables"] == 13 and info["bus_pitch"] % 16 == 0
    # a closed screen is dead and out of the cache (use after free)
    scr.close()
    with pytest.raises(ValueError):
        scr.run(inj, tol)
    scr2 = screen.screen_for(ptdf, inst)
    assert scr2 is not scr and scr2.handle is not None
    scr2.run(inj, tol)
    np.testing.assert_allclose(scr2.flows(0), g["c3_tables"][0] @ inj, rtol=0,
                               atol=1e-12 * max(1.0, np.abs(g["c3_tables"][0] @ inj).max()))


@pytest.mark.gpu
def test_device_screen_sizes_and_edges():
    """Large random tables (ragged line/bus counts, T = 24/36/1/96, split bus
    range) against numpy; tol = 0 and an all-clear screen."""
    rng = np.random.default_rng(4)
    for n_l, n_b, n_t in ((1, 1, 1), (300, 17, 24), (1031, 2049, 36), (129, 4000, 96)):
        tab = rng.standard_normal((n_l, n_b)) * 0.2
        inj = rng.standard_normal((n_b, n_t)) * 50
        lim = np.abs(rng.standard_normal(n_l)) * 40 + 1
        lines = [_Line({"id": f"l{i}", "limit": lim[i], "emergency_limit": lim[i]})
                 for i in range(n_l)]
        scr = screen.FlowScreen(_Ptdf(["base"], [tab]), ["base"], lines)
        for tol in (0.0, 1e-4):
            tb, li, pe, fl, ex = scr.run(inj, tol)
            flows = tab @ inj
            np.testing.assert_allclose(scr.flows(0), flows, rtol=0,
                                       atol=1e-12 * max(1.0, np.abs(tab).sum(1).max() * 200))
            want = np.abs(flows) - lim[:, None]
            sure = want > tol * lim[:, None] + 1e-9 * (1 + np.abs(flows))
            maybe = want > tol * lim[:, None] - 1e-9 * (1 + np.abs(flows))
            got = np.zeros_like(sure)
            got[li, pe] = True
            assert not (sure & ~got).any() and not (got & ~maybe).any()
            assert (tb == 0).all() and len(np.unique(li * n_t + pe)) == len(li)
        tb, *_ = scr.run(inj * 0.0, 1e-4)
        assert len(tb) == 0
        scr.close()
    # a horizon longer than one launch (200 periods) runs in period chunks
    tab = rng.standard_normal((70, 50)) * 0.2
    inj = rng.standard_normal((50, 200)) * 50
    lim = np.full(70, 30.0)
    lines = [_Line({"id": f"l{i}", "limit": 30.0, "emergency_limit": 30.0}) for i in range(70)]
    scr = screen.FlowScreen(_Ptdf(["base"], [tab]), ["base"], lines)
    tb, li, pe, fl, ex = scr.run(inj, 0.0)
    flows = tab @ inj
    want = set(zip(*np.nonzero(np.abs(flows) - lim[:, None] > 1e-9)))
    got = set(zip(li.tolist(), pe.tolist()))
    assert want <= got and pe.max() >= 96
    np.testing.assert_allclose(fl, flows[li, pe], rtol=0, atol=1e-9)
    scr.close()


def _scuckit():
    import sys
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "scuckit")) and p not in sys.path:
            sys.path.append(p)
    try:
        import scuckit  # noqa: F401
        return True
    except Exception:
        return False


@pytest.mark.gpu
@pytest.mark.skipif(not _scuckit(), reason="reference package not installed")
def test_install_routes_driver_screen():
    """After hprlp.install() the driver's name lookup (driver.py:288) reaches
    the device screen, which takes the reference's own ScucInstance and
    PtdfTable (read-only arrays) and returns its Violation class."""
    import scuckit
    import scuckit.driver as drv
    from scuckit import compute_ptdf, parse_instance
    from paper_2510_10891_b200 import hprlp, scuc
    ref_fn = drv.screen_violations
    doc = scuc.generate_instance(30, 10, 41, 24, seed=9, n_contingencies=6)
    inst = parse_instance(doc)
    ptdf = compute_ptdf(inst.network)
    u, pp, pen, n_cols = screen.column_blocks(inst)
    rng = np.random.default_rng(2)
    x = np.zeros(n_cols)
    x[u] = 1.0
    x[pp] = rng.uniform(0, 1, size=u.shape) * np.array(
        [[g.p_max - g.p_min] for g in inst.generators])
    want = ref_fn(x, inst, ptdf, tol=1e-4)
    hprlp.install()
    try:
        assert drv.screen_violations is screen.screen_violations
        assert scuckit.screen_violations is screen.screen_violations
        got = drv.screen_violations(x, inst, ptdf, tol=1e-4)
        assert all(type(v) is drv.Violation for v in got)
    finally:
        hprlp.uninstall()
    assert drv.screen_violations is ref_fn
    ref = [[v.line, v.period, v.contingency, v.flow, v.limit, v.excess, v.already_monitored]
           for v in want]
    tabs = np.stack([ptdf.table(k) for k in inst.contingency_keys()])
    _compare(got, ref, tabs, screen.injections(x, inst))


def _oracle_run(ci):
    """A shard's records from numpy products (stands in for the device screen
    in the CPU gloo test; the merge and ordering are what is under test)."""
    g = golden()
    _, inst, _, _ = case(g, ci)
    keys = inst.contingency_keys()
    tabs, lims = g[f"c{ci}_tables"], g[f"c{ci}_limits"]

    def run(mine, inj, tol):
        out = [[], [], [], [], []]
        for j, key in enumerate(mine):
            k = keys.index(key)
            flows = tabs[k] @ inj
            ex = np.abs(flows) - lims[k][:, None]
            li, pe = np.nonzero(ex > tol * lims[k][:, None])
            for a, v in zip(out, (np.full(li.size, j), li, pe, flows[li, pe], ex[li, pe])):
                a.append(v)
        return tuple(np.concatenate(a).astype(t) for a, t in
                     zip(out, (np.int32, np.int32, np.int32, np.float64, np.float64)))
    return run


def _shard_worker(rank, ws, port, ci, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        g = golden()
        _, inst, ptdf, tol = case(g, ci)
        res = []
        for x, mon, _ in points(g, ci):
            got = screen.screen_violations_sharded(x, inst, ptdf, monitored=mon, tol=tol,
                                                   _run=_oracle_run(ci))
            res.append([[v.line, v.period, v.contingency, v.flow, v.limit, v.excess,
                         v.already_monitored] for v in got])
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_sharded_screen_gloo_matches_reference(ws):
    """Keys sharded round robin over ws gloo ranks; every rank returns the
    reference's exact list (golden case 3: 13 keys)."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, ws, port, 3, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    refs = [r for _, _, r in points(golden(), 3)]
    for _, res in out:
        assert res == refs
    assert screen.shard_keys(list("abcde"), 2, 1) == ["b", "d"]


@pytest.mark.gpu
def test_sharded_screen_single_rank_device():
    """The sharded entry with its device screen (one rank, gloo group)."""
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        g = golden()
        doc, inst, ptdf, tol = case(g, 1)
        for x, mon, ref in points(g, 1):
            got = screen.screen_violations_sharded(x, inst, ptdf, monitored=mon, tol=tol, device=0)
            _compare(got, ref, g["c1_tables"], screen.injections(x, inst))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_fp64_peak_probe_is_plausible():
    """The measured DMMA ceiling the bench's screen roofline divides by."""
    v = screen.fp64_peak_tflops()
    assert 5.0 < v < 100.0


@pytest.mark.gpu
def test_nonfinite_point_matches_oracle():
    """A NaN or inf in the point makes that period's flows non-finite; as in
    the reference, NaN excesses never pass the test and +inf ones do."""
    g = golden()
    doc, inst, ptdf, tol = case(g, 0)
    keys = inst.contingency_keys()
    u, pp, pen, _ = screen.column_blocks(inst)
    for bad in (np.nan, np.inf):
        x = g["c0_p0_x"].copy()
        x[pp[0, 3]] = bad
        got = screen.screen_violations(x, inst, ptdf, tol=tol)
        want = screen_oracle.screen(g["c0_tables"], g["c0_limits"], keys,
                                    [ln.lid for ln in inst.lines], oracle_inj(doc, inst, x), (), tol)
        assert {v.triple for v in got} == {w[:3] for w in want}
        assert not any(v.period == 3 for v in got) or bad == np.inf
