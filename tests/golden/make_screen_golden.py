"""Golden flow-screen vectors from the UNMODIFIED reference (build container
only):  python tests/golden/make_screen_golden.py

For seeded instances (with single-line contingencies) the reference's
parse_instance + compute_ptdf (instance.py:241-268) build the PTDF tables and
its screen_violations (driver.py:165-200) screens seeded points.  Saved to
tests/golden/screen.npz: the instance document, the tables, the per-key
limits, the points and the reference's violation lists.  tests/test_screen.py
pins oracle/screen_oracle.py on them (CPU) and checks the device screen
against them (GPU box, no reference checkout needed there)."""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from scuckit import compute_ptdf, parse_instance  # noqa: E402
from scuckit.driver import screen_violations  # noqa: E402
from scuckit.formulation import VariableMap  # noqa: E402

from paper_2510_10891_b200 import scuc  # noqa: E402

# (buses, gens, lines, periods, seed, contingencies, tol)
CASES = [(14, 6, 20, 24, 3, 5, 1e-4), (30, 10, 41, 36, 7, 8, 1e-4), (57, 16, 80, 24, 11, 0, 0.0),
         (118, 30, 186, 36, 1, 12, 1e-3)]
POINTS = 3


def seeded_point(inst, vmap, rng, scale):
    x = np.zeros(vmap.n_cols)
    on = (rng.random(vmap.u.shape) < 0.7).astype(float)
    x[vmap.u] = on
    pmax = np.array([[g.p_max - g.p_min] for g in inst.generators])
    x[vmap.pprime] = on * pmax * rng.random(vmap.u.shape) * scale
    x[vmap.penalty] = rng.random(vmap.penalty.shape) * 5.0 * (rng.random(vmap.penalty.shape) < 0.1)
    return x


if __name__ == "__main__":
    out = {}
    for ci, (nb, ng, nl, nt, seed, nc, tol) in enumerate(CASES):
        doc = scuc.generate_instance(nb, ng, nl, nt, seed=seed, n_contingencies=nc)
        inst = parse_instance(doc)
        ptdf = compute_ptdf(inst.network)
        vmap = VariableMap(inst)
        keys = inst.contingency_keys()
        out[f"c{ci}_doc"] = np.array(json.dumps(doc))
        out[f"c{ci}_tables"] = np.stack([ptdf.table(k) for k in keys])
        out[f"c{ci}_limits"] = np.array([[ln.limit_for(k) for ln in inst.lines] for k in keys])
        out[f"c{ci}_tol"] = np.array(tol)
        rng = np.random.default_rng(100 + ci)
        for p in range(POINTS):
            x = seeded_point(inst, vmap, rng, scale=0.6 + 0.4 * p)
            lids = [ln.lid for ln in inst.lines]
            monitored = {(lids[i], t, keys[0]) for i in range(0, len(lids), 3) for t in (0, 5)}
            viol = screen_violations(x, inst, ptdf, monitored=monitored, tol=tol)
            out[f"c{ci}_p{p}_x"] = x
            out[f"c{ci}_p{p}_monitored"] = np.array(json.dumps(sorted(monitored)))
            out[f"c{ci}_p{p}_viol"] = np.array(json.dumps(
                [[v.line, v.period, v.contingency, v.flow, v.limit, v.excess,
                  v.already_monitored] for v in viol]))
            print(f"case {ci} point {p}: {len(viol)} violations over {len(keys)} keys")
    np.savez_compressed(os.path.join(HERE, "screen.npz"), **out)
