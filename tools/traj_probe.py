"""Trajectory diffs of the engine against the committed reference records
(tests/golden/c1_trajectory.json, c2_trajectory.json, c4_window.json): the
numbers the hardened parity tests' tolerances are set from.

    python tools/traj_probe.py [--out gpurun_out/traj_probe.json] [--c4]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_10891_b200 import hprlp, scuc  # noqa: E402
from paper_2510_10891_b200.lp import Precision  # noqa: E402
from tests import golden_io  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--c4", action="store_true")
ap.add_argument("--c4full", action="store_true", help="also the full C4 runs (c4_full_*.json)")
a = ap.parse_args()


def first_over(byrow, tol):
    bad = [i for i, v in enumerate(byrow) if v > tol]
    return bad[0] if bad else len(byrow)


def probe(name, lpa, gg, prec, max_it=None):
    cfg = dict(tolerance=1e-4, ruiz=False, precision=Precision(prec), log_residuals=True)
    if max_it:
        cfg["max_iterations"] = max_it
    t = time.perf_counter()
    r = hprlp.solve(lpa.to_lp(), hprlp.SolverConfig(**cfg))
    wall = time.perf_counter() - t
    mine, ref = golden_io.log_rows(r), np.array(gg["log"])
    d = golden_io.trajectory_diff(mine, ref)
    rm, rr = golden_io.restart_list(mine), golden_io.restart_list(ref)
    byrow = d.pop("max_rel_by_row")
    out = dict(name=name, prec=prec, wall_s=wall, status=(r.status.value, gg["status"]),
               iterations=(r.iterations, gg["iterations"]), restarts=(r.restarts, gg["restarts"]),
               lam_rel=abs(r.lam - gg["lam"]) / gg["lam"],
               obj_rel=abs(r.objective - gg["objective"]) / abs(gg["objective"]),
               restart_iters_equal=[x[0] for x in rm] == [x[0] for x in rr],
               restart_kinds_equal=[x[1] for x in rm] == [x[1] for x in rr],
               sigma_after_max_rel=max([abs(x[3] - y[3]) / y[3] for x, y in zip(rm, rr)],
                                       default=0.0),
               rows_within_1e5=first_over(byrow, 1e-5), rows_within_1e9=first_over(byrow, 1e-9),
               worst_row=int(np.argmax(byrow)) if byrow else -1, **d)
    print(json.dumps(out), flush=True)
    return out


res = []
doc, mon, lpa = scuc.build_config("C1")
g = golden_io.c1()
print("C1 digest", lpa.digest() == g["digest"], flush=True)
res.append(probe("C1", lpa, g["fp64"], "fp64"))
res.append(probe("C1", lpa, g["fp32"], "fp32"))
doc, mon, lpa = scuc.build_config("C2", n_triples=500)
g = golden_io.c2()
print("C2 digest", lpa.digest() == g["digest"], flush=True)
res.append(probe("C2", lpa, g["fp64"], "fp64"))
if a.c4:
    g = golden_io.c4_window()
    doc, mon, lpa = scuc.build_config("C4")
    print("C4 digest", lpa.digest() == g["digest"], flush=True)
    for prec in ("fp64", "fp32"):
        o = probe("C4-window", lpa, g[prec], prec, max_it=g["max_iterations"])
        res.append(o)
if a.c4full:
    doc, mon, lpa = scuc.build_config("C4")
    for prec in ("fp64", "fp32"):
        p = os.path.join(golden_io.GOLDEN, f"c4_full_{prec}.json")
        if os.path.exists(p):
            g = json.load(open(p))
            print("C4 full digest", lpa.digest() == g["digest"], flush=True)
            res.append(probe("C4-full", lpa, g[prec], prec))
if a.out:
    with open(a.out, "w") as fh:
        json.dump(res, fh, indent=1)
