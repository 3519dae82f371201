"""C5 on one B200: build the N-1 LP (C4 + 20,000 contingency flow triples via
LODF rows), upload it, and run a fixed window of HPR iterations.  Prints one
JSON line with the build / engine / setup / loop timings and the layout.

    python tools/c5_probe.py [--triples 20000] [--iters 256] [--partitioned]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_10891_b200 import hprlp, scuc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--triples", type=int, default=20000)
ap.add_argument("--iters", type=int, default=256)
ap.add_argument("--partitioned", action="store_true")
a = ap.parse_args()

out = {"config": "C5", "triples": a.triples}
t = time.perf_counter()
doc, mon, lpa = scuc.build_config("C5", n_triples=a.triples)
out["build_s"] = time.perf_counter() - t
out["shape"], out["nnz"] = list(lpa.shape), lpa.nnz
print(json.dumps(out), flush=True)
lp = lpa.to_lp()
cfg = hprlp.SolverConfig(tolerance=1e-4, ruiz=False, max_iterations=a.iters, log_residuals=True)
t = time.perf_counter()
if a.partitioned:
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("gloo", rank=0, world_size=1)
    r = hprlp.solve_partitioned(lp, cfg)
else:
    eng = hprlp.Engine(lp)
    out["engine_s"] = time.perf_counter() - t
    out["workspace_gb"] = eng.workspace_bytes / 1e9
    out["layout"] = eng.layout()
    t = time.perf_counter()
    r = hprlp._solve_once(lp, cfg, None, time.perf_counter(), engine=eng)
out["solve_s"] = time.perf_counter() - t
ds = getattr(r, "device_stats", {})
out.update(status=r.status.value, iterations=r.iterations, restarts=r.restarts,
           objective=r.objective, lam=r.lam, loop_s=ds.get("loop_seconds"),
           setup_s=ds.get("setup_seconds"),
           it_per_s=(r.iterations / ds["loop_seconds"]) if ds.get("loop_seconds") else None,
           first_rows=[[e["iteration"], e["rel_primal"], e["rel_dual"], e["rel_gap"]]
                       for e in r.residual_log[:4]],
           max_mem_gb=torch.cuda.max_memory_allocated() / 1e9)
print(json.dumps(out), flush=True)
