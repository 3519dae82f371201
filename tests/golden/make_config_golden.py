"""Golden solves of the UNMODIFIED reference under non-default SolverConfig
fields (build container only):

    python tests/golden/make_config_golden.py

Eight random LPs of tests/golden/random_lps.npz are solved by
scuckit.hprlp.solve under seven config variants that move every field the
driver never touches (check_every, restart_beta / restart_stall,
sigma0, sigma_damping, ruiz_iters, pock_chambolle, normalize_rhs_objective,
power_tol / power_inflation / power_max_iter, seed, max_iterations).  The
record per (LP, variant) is written to tests/golden/config_variants.json;
tests/test_oracle_golden.py pins the oracle to it and
tests/test_gpu_parity.py pins the engine."""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from scuckit import hprlp  # noqa: E402
from scuckit.lp_kernel import SparseMatrix, StandardFormLp  # noqa: E402

from tests import golden_io  # noqa: E402

VARIANTS = {
    "cadence": dict(tolerance=1e-7, check_every=8, restart_beta=0.3, restart_stall=100),
    "sigma": dict(tolerance=1e-7, sigma0=0.7, sigma_damping=0.3, ruiz_iters=3),
    "no_pc_no_norm": dict(tolerance=1e-7, pock_chambolle=False, normalize_rhs_objective=False),
    "power": dict(tolerance=1e-7, power_tol=1e-6, power_inflation=1.05, power_max_iter=200,
                  seed=7),
    "bare": dict(tolerance=1e-7, ruiz=False, pock_chambolle=False, check_every=32),
    "iter_limit": dict(tolerance=1e-12, max_iterations=500),
    "tail_only": dict(tolerance=1e-12, max_iterations=10, check_every=16),
    "long_cadence": dict(tolerance=1e-7, check_every=100, restart_stall=1000),
}
KEYS = ("iterations", "restarts", "objective", "lam", "sigma_final")


def ref_lp(lp):
    return StandardFormLp(matrix=SparseMatrix(lp.matrix.csr), rhs=lp.rhs, cost=lp.cost,
                          lower=lp.lower, upper=lp.upper, n_eq=lp.n_eq, offset=lp.offset)


if __name__ == "__main__":
    out = {}
    lps = golden_io.random_lps()[:8]
    for i, (lp, _, _) in enumerate(lps):
        for name, kw in VARIANTS.items():
            r = hprlp.solve(ref_lp(lp), hprlp.SolverConfig(**kw))
            rec = {k: float(getattr(r, k)) for k in KEYS}
            rec["status"] = r.status.value
            out[f"{i}/{name}"] = rec
    with open(os.path.join(HERE, "config_variants.json"), "w") as fh:
        json.dump({"variants": VARIANTS, "results": out}, fh, indent=0)
    print(len(out), sorted({v["status"] for v in out.values()}))
