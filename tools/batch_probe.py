"""Overlapped small-LP solves: K cost-perturbed copies of
a C1/C2-size LP, solved one after another with hprlp.solve and all at once
with hprlp.solve_many; prints one JSON line with both wall times.

    python tools/batch_probe.py [--config C1] [--copies 8] [--tol 1e-4]"""

import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_10891_b200 import hprlp, scuc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--copies", type=int, default=8)
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--workers", type=int, default=8)
    a = ap.parse_args()
    doc, mon, lpa = scuc.build_config(a.config)
    rng = np.random.default_rng(0)
    lps = []
    for _ in range(a.copies):
        lp = lpa.to_lp()                      # its own matrix object, as each node LP has
        lps.append(dataclasses.replace(
            lp, cost=lp.cost * (1.0 + 0.01 * rng.random(lp.cost.size))))
    cfg = hprlp.SolverConfig(tolerance=a.tol, ruiz=False)
    hprlp.solve(lps[0], cfg)                          # warm the library / context
    t0 = time.perf_counter()
    seq = [hprlp.solve(lp, cfg) for lp in lps]
    t_seq = time.perf_counter() - t0
    t0 = time.perf_counter()
    par = hprlp.solve_many(lps, cfg, workers=a.workers)
    t_par = time.perf_counter() - t0
    same = all(p.iterations == s.iterations and p.objective == s.objective
               for p, s in zip(par, seq))
    print(json.dumps({"config": a.config, "lp": list(lpa.shape), "nnz": lpa.nnz,
                      "copies": a.copies, "workers": a.workers, "tol": a.tol,
                      "iterations": [r.iterations for r in seq],
                      "sequential_s": t_seq, "overlapped_s": t_par,
                      "speedup": t_seq / t_par, "identical_results": same}))


if __name__ == "__main__":
    main()
