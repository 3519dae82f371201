"""Golden presolve digests from the UNMODIFIED reference (build container
only):  python tests/golden/make_presolve_golden.py

For each seeded case of tests/presolve_cases.py the reference's
milp_presolve (presolve.py:212-257) and, when feasible, lp_presolve of the
relaxation (:260-288) run on the reference's own classes; the digests of
(reduced model, ReductionLog) go to tests/golden/presolve.json.
tests/test_presolve.py recomputes them with the native-core mirror on this
package's classes (the GPU box has no reference checkout)."""

import json
import os
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from scuckit import presolve  # noqa: E402
from scuckit.formulation import MilpModel  # noqa: E402
from scuckit.lp_kernel import SparseMatrix, StandardFormLp  # noqa: E402

from tests.presolve_cases import digest, random_case  # noqa: E402

N_CASES = 60

if __name__ == "__main__":
    cls = types.SimpleNamespace(SparseMatrix=SparseMatrix, StandardFormLp=StandardFormLp,
                                MilpModel=MilpModel)
    out = {}
    for seed in range(N_CASES):
        model, kind = random_case(seed, cls)
        red, log = presolve.milp_presolve(model)
        rec = {"kind": kind, "milp": digest((red, log)), "infeasible": log.infeasible}
        if log.feasible:
            res = presolve.lp_presolve(red.relax())
            rec["lp"] = digest(res)
            rec["lp_infeasible"] = res[1].infeasible
        out[str(seed)] = rec
    with open(os.path.join(HERE, "presolve.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    kinds = [r["infeasible"].split(" ")[0] if r["infeasible"] else "feasible" for r in out.values()]
    print({k: kinds.count(k) for k in set(kinds)})
