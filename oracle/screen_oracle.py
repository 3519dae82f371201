"""CPU oracle of the post-MILP flow screen — TEST INFRASTRUCTURE ONLY.

Restates ``scuckit.driver.screen_violations`` (``pkg/src/scuckit/driver.py:165-200``)
on plain arrays so the device screen (``paper_2510_10891_b200/screen.py``) can be
checked without the reference installed.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU legs may import it.  Pinned against the reference's own
output by ``tests/golden/screen.npz`` (``tests/golden/make_screen_golden.py``).
"""

from __future__ import annotations

import numpy as np


def injections(point, n_gens, n_periods, n_buses, seg_total, p_min, gen_bus, demand):
    """driver.py:176-181 with VariableMap's column layout (formulation.py:53-70):
    u at 0, p' at 3GT, penalty after 4GT + T*sum(H) + GT."""
    gt = n_gens * n_periods
    u = np.arange(gt).reshape(n_gens, n_periods)
    pprime = 3 * gt + u
    pen0 = 4 * gt + n_periods * seg_total + gt
    penalty = pen0 + np.arange(n_buses * n_periods).reshape(n_buses, n_periods)
    point = np.asarray(point, dtype=np.float64)
    power = point[pprime] + np.asarray(p_min, dtype=np.float64).reshape(-1, 1) * point[u]
    inj = -(np.asarray(demand, dtype=np.float64) - point[penalty])
    for gi in range(n_gens):                                    # driver.py:180-181
        inj[gen_bus[gi], :] += power[gi, :]
    return inj


def screen(tables, limits, keys, line_ids, inj, monitored=(), tol=1e-4):
    """driver.py:184-200: (line, period, contingency, flow, limit, excess,
    already_monitored) tuples sorted by (-excess, line, period, contingency)."""
    monitored = set(monitored)
    out = []
    for k, key in enumerate(keys):
        flows = tables[k] @ inj                                 # driver.py:186
        for li, lid in enumerate(line_ids):
            limit = float(limits[k][li])                        # Line.limit_for
            for t in range(inj.shape[1]):
                excess = abs(flows[li, t]) - limit
                if excess > tol * limit:
                    out.append((lid, t, key, float(flows[li, t]), limit, float(excess),
                                (lid, t, key) in monitored))
    out.sort(key=lambda v: (-v[5], v[0], v[1], v[2]))
    return out
