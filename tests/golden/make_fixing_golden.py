"""Golden successive-fixing record from the UNMODIFIED reference (build
container only):  PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_fixing_golden.py

Runs scuckit.successive_fixing (fixing.py:142-186) with the reference CPU HPR
solver (SolverConfig(tolerance=1e-4, ruiz=False), the driver's fixing-loop
settings, driver.py:54,61-65) on the C1-structure instance with instance
scaling and all base flow triples, and records per round the presolved LP
digest, the LP objective / iterations, and the final fixed-column ledger.
tests/test_dropin_fixing.py replays the same loop with the GPU engine
install()ed and compares (parity criterion of the north star: identical
fixed sets wherever no relaxed binary is within 1e-6 of a threshold)."""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from scuckit import (apply_instance_scaling, build_model, hprlp, lp_backends,  # noqa: E402
                     parse_instance, successive_fixing)

from paper_2510_10891_b200 import scuc  # noqa: E402


def lp_digest(lp):
    c = lp.matrix.csr
    h = hashlib.sha256()
    for a in (c.indptr.astype(np.int64), c.indices.astype(np.int64), c.data, lp.rhs, lp.cost,
              lp.lower, lp.upper):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run(doc, rounds=2, tau=0.1):
    inst, _ = apply_instance_scaling(parse_instance(doc))
    model, _ = build_model(inst, monitored=scuc.all_base_triples(doc))
    cfg = hprlp.SolverConfig(tolerance=1e-4, ruiz=False)
    rec = []

    def solver(lp):
        r = lp_backends.solve_lp(lp, "hpr", cfg)
        rec.append({"digest": lp_digest(lp), "shape": list(lp.matrix.shape),
                    "objective": r.objective, "iterations": r.iterations, "status": r.status})
        return r

    t = time.time()
    error = None
    try:
        successive_fixing(model, rounds, solver, tau)   # fixes accumulate on `model`
    except Exception as exc:                             # e.g. InfeasibleModelError
        error = f"{type(exc).__name__}: {exc}"
    return {"rounds": rec, "fixed": {str(k): v.value for k, v in sorted(model.fixed.items())},
            "error": error, "seconds": time.time() - t}


if __name__ == "__main__":
    doc = scuc.generate_instance(**scuc.CONFIGS["C1"])
    res = run(doc)
    print(len(res["fixed"]), [(r["iterations"], r["objective"]) for r in res["rounds"]],
          res["seconds"])
    with open(os.path.join(HERE, "c1_fixing.json"), "w") as fh:
        json.dump(res, fh)
