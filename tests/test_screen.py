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
import types

import numpy as np
import pytest

from oracle import screen_oracle
from paper_2510_10891_b200 import screen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "screen.npz")
N_CASES, N_POINTS = 4, 3


def golden():
    return np.load(GOLD)


class _Line:
    def __init__(self, d):
        self.lid, self.limit, self.emergency_limit = d["id"], d["limit"], d["emergency_limit"]

    def limit_for(self, key):                      # instance.py:88-89
        return self.limit if key == "base" else self.emergency_limit


def instance_of(doc):
    """The attributes screen_violations reads from a ScucInstance
    (instance.py:99-139), built from the golden document."""
    gens = tuple(types.SimpleNamespace(gid=g["id"], bus=g["bus"], p_min=g["p_min"],
                                       n_segments=len(g["segments"])) for g in doc["generators"])
    buses = tuple(types.SimpleNamespace(bid=b["id"], demand=b["demand"]) for b in doc["buses"])
    lines = tuple(_Line(ln) for ln in doc["lines"])
    conts = tuple(types.SimpleNamespace(cid=c["id"]) for c in doc["contingencies"])
    net = types.SimpleNamespace(buses=buses, lines=lines, contingencies=conts,
                                bus_index=lambda: {b.bid: i for i, b in enumerate(buses)})
    return types.SimpleNamespace(
        generators=gens, buses=buses, lines=lines, contingencies=conts, network=net,
        n_periods=doc["time_periods"],
        demand_matrix=lambda: np.array([b.demand for b in buses], dtype=np.float64),
        contingency_keys=lambda: ["base"] + [c.cid for c in conts])


class _Ptdf:
    """PtdfTable's read interface (instance.py:141-173) over the golden tables."""

    def __init__(self, keys, tables):
        self._t = dict(zip(keys, tables))

    def table(self, key="base"):
        return self._t[key]


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
