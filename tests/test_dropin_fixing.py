"""Drop-in check: the reference's successive fixing (scuckit.fixing, Alg. 2)
with its LP solves routed to the B200 engine by ``hprlp.install()``.

Needs the reference package importable: the build container's
/root/reference, or the ``baseline/_ref`` install that travels to the GPU
box (``pip install --no-deps --target baseline/_ref <reference pkg>``).  The
north-star criterion: identical fixed-variable sets wherever no relaxed
binary lies within 1e-6 of a fixing threshold, and LP objectives within the
solver tolerance.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _scuckit():
    for p in (REF, "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "scuckit")) and p not in sys.path:
            sys.path.append(p)
    try:
        import scuckit  # noqa: F401
        return True
    except Exception:
        return False


pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not _scuckit(), reason="reference package not installed")]


def _fixing_run(doc, rounds=2, tau=0.1):
    from scuckit import (apply_instance_scaling, build_model, hprlp, lp_backends,
                         parse_instance, successive_fixing)
    from paper_2510_10891_b200 import scuc
    inst, _ = apply_instance_scaling(parse_instance(doc))
    model, _ = build_model(inst, monitored=scuc.all_base_triples(doc))
    cfg = hprlp.SolverConfig(tolerance=1e-4, ruiz=False)
    rec = []

    def solver(lp):
        r = lp_backends.solve_lp(lp, "hpr", cfg)
        rec.append((r.objective, r.iterations, r.status, r.x))
        return r

    error = None
    try:
        successive_fixing(model, rounds, solver, tau)    # fixes accumulate on `model`
    except Exception as exc:                              # e.g. InfeasibleModelError
        error = f"{type(exc).__name__}: {exc}"
    return rec, {k: v.value for k, v in model.fixed.items()}, error


def _near_threshold(x, tau, tol=1e-6):
    x = np.asarray(x)
    return bool(np.any((np.abs(x - tau) < tol) | (np.abs(x - (1 - tau)) < tol)))


def _assert_fixed_sets(recs, tau, got, want, what):
    """The north-star fixed-set criterion: identical sets unless a relaxed
    value lies within 1e-6 of a fixing threshold.  A skipped comparison is
    reported (warning + stdout), never silent."""
    import warnings
    near = [i for i, r in enumerate(recs) if _near_threshold(r[3], tau)]
    if near:
        msg = (f"{what}: fixed-set assertion skipped -- round(s) {near} have a relaxed "
               f"value within 1e-6 of tau={tau}")
        print(msg)
        warnings.warn(msg)
        return False
    assert got == want
    return True


def test_successive_fixing_gpu_matches_cpu():
    """Small instance: the reference loop twice on the box, CPU HPR vs GPU."""
    import scuckit.hprlp as ref_hprlp
    from paper_2510_10891_b200 import hprlp as gpu, scuc
    doc = scuc.generate_instance(30, 12, 45, 8, seed=3)
    cpu_rec, cpu_fixed, cpu_err = _fixing_run(doc)
    gpu.install()
    try:
        assert ref_hprlp.solve is gpu.solve
        gpu_rec, gpu_fixed, gpu_err = _fixing_run(doc)
    finally:
        gpu.uninstall()
    assert ref_hprlp.solve is not gpu.solve
    assert len(gpu_rec) == len(cpu_rec)
    for (oc, ic, sc, xc), (og, ig, sg, xg) in zip(cpu_rec, gpu_rec):
        assert sc == sg == "optimal-tolerance"
        assert abs(og - oc) <= 1e-6 * abs(oc)
    _assert_fixed_sets(cpu_rec, 0.1, (gpu_fixed, gpu_err), (cpu_fixed, cpu_err),
                       "30-bus GPU vs CPU")


def test_successive_fixing_c1_against_reference_record():
    """C1 structure (118 buses, 54 units, 24 periods, all base flow rows):
    the GPU-driven fixing loop against the reference's own CPU record
    (tests/golden/c1_fixing.json, produced by make_fixing_golden.py)."""
    path = os.path.join(ROOT, "tests", "golden", "c1_fixing.json")
    if not os.path.exists(path):
        pytest.skip("c1_fixing.json not generated")
    g = json.load(open(path))
    import scuckit.hprlp as ref_hprlp
    from paper_2510_10891_b200 import hprlp as gpu, scuc
    doc = scuc.generate_instance(**scuc.CONFIGS["C1"])
    gpu.install()
    try:
        rec, fixed, err = _fixing_run(doc)
    finally:
        gpu.uninstall()
    assert len(rec) == len(g["rounds"])
    for (og, ig, sg, xg), r in zip(rec, g["rounds"]):
        assert sg == r["status"]
        assert abs(og - r["objective"]) <= 1e-6 * abs(r["objective"])
    want = {int(k): v for k, v in g["fixed"].items()}
    _assert_fixed_sets(rec, 0.1, (fixed, err), (want, g["error"]), "C1 vs reference record")


def _report(rep):
    d = rep.to_json_dict()
    d.pop("timings")
    return d


def _assert_same_run(got, want, what):
    assert got["status"] == want["status"] == "solved", what
    assert got["exit_code"] == want["exit_code"]
    assert abs(got["objective"] - want["objective"]) <= 1e-9 * abs(want["objective"]), what
    assert got["monitored"] == want["monitored"]
    assert got.get("commitment") == want.get("commitment")
    assert got["fixing"] == want["fixing"]
    assert got["nodes_total"] == want["nodes_total"]
    assert len(got["passes"]) == len(want["passes"])
    for a, b in zip(got["passes"], want["passes"]):
        for k in ("stage", "index", "monitored_rows", "free_binaries", "milp_status",
                  "milp_nodes", "violations_found"):
            assert a[k] == b[k], (what, k, a[k], b[k])
        assert abs(a["milp_gap"] - b["milp_gap"]) <= 1e-5


def test_driver_run_completes_like_reference():
    """North-star end-to-end criterion: the reference's own two-stage driver
    (driver.run, driver.py:203-324) run to completion on a small instance,
    once on its CPU path and once with install() routing LP solves, presolve,
    the flow screen and the model builder to this package.  Same final MILP
    objective (HiGHS-polished incumbent, milp_bb.py:146-162), commitment,
    monitored set, fixing record per round, B&B nodes and pass records -- also
    against the reference's record from the build container
    (tests/golden/sf_small.json, make_sf_golden.py)."""
    from scuckit import driver, parse_instance
    from paper_2510_10891_b200 import hprlp as gpu, scuc
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "sf_small.json")))
    doc = scuc.generate_instance(**g["instance"])
    cpu = _report(driver.run(parse_instance(doc), driver.DriverConfig(time_limit=600.0)))
    gpu.install()
    try:
        got = _report(driver.run(parse_instance(doc), driver.DriverConfig(time_limit=600.0)))
    finally:
        gpu.uninstall()
    _assert_same_run(cpu, g["report"], "reference on the box vs its record")
    _assert_same_run(got, cpu, "B200 path vs reference on the box")


def test_speculative_bb_leaves_the_search_unchanged():
    """bb.py: the plunge's waiting sibling is solved ahead on a second engine
    and stream; the reference's B&B (milp_bb.py:279-404) must take exactly the
    same path -- node log, incumbent, bound, node and LP-solve counts -- as
    with speculation off, and the speculative results must actually be used."""
    from scuckit import apply_instance_scaling, build_model, parse_instance
    from scuckit.milp_bb import BbConfig, solve_milp
    from scuckit.presolve import milp_presolve
    from paper_2510_10891_b200 import bb, hprlp as gpu, scuc
    doc = scuc.generate_instance(30, 12, 45, 8, seed=3, shutdown_feasible=True)
    inst, _ = apply_instance_scaling(parse_instance(doc))
    out = {}
    for spec in (False, True):
        gpu.install(bb=spec)            # opt-in (install() leaves the B&B as written)
        try:
            model, _ = build_model(inst, monitored=scuc.sample_monitored(doc, 40, 3))
            red, log = milp_presolve(model)
            before = dict(bb.STATS)
            res = solve_milp(red, gap=1e-4, config=BbConfig(node_limit=40))
            out[spec] = (res, {k: bb.STATS[k] - before[k] for k in bb.STATS})
        finally:
            gpu.uninstall()
    (a, _), (b, st) = out[False], out[True]
    assert (a.status, a.nodes, a.lp_solves) == (b.status, b.nodes, b.lp_solves)
    assert a.objective == b.objective or (np.isnan(a.objective) and np.isnan(b.objective))
    assert a.bound == b.bound
    assert [(n["node"], n["action"], n["bound"]) for n in a.node_log] == \
           [(n["node"], n["action"], n["bound"]) for n in b.node_log]
    print("speculation", st)
    assert st["speculated"] > 0 and st["hits"] > 0
