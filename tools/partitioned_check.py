"""Multi-rank check of the row-partitioned engine, one GPU
per rank over NCCL, launched by torchrun:

    torchrun --standalone --nproc-per-node 2 tools/partitioned_check.py

Every rank builds the same C2 + 500-triple LP (flow panels live), rank 0 also
solves it on one GPU alone, and each rank then runs ``hprlp.solve_partitioned``
(A row-partitioned by period, A^T y partials all-reduced over NCCL inside the
block graph, replicated controller, device-side stop flag).  Rank 0 checks the
partitioned solve against the single-GPU one and prints one JSON line; exit
code 0 means every check held on every rank.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2510_10891_b200 import hprlp, scuc  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")          # bootstrap only; the solve runs over NCCL
    rank, ws = dist.get_rank(), dist.get_world_size()
    doc, mon, lpa = scuc.build_config("C2", n_triples=500)
    lp = lpa.to_lp()
    cfg = hprlp.SolverConfig(tolerance=1e-4, ruiz=False, log_residuals=True)
    ref = hprlp.solve(lp, cfg) if rank == 0 else None
    comm = hprlp.NcclComm(device=local)
    try:
        r = hprlp.solve_partitioned(lp, cfg, comm=comm)
        tl = hprlp.solve_partitioned(lp, hprlp.SolverConfig(tolerance=1e-12, time_limit=0.5,
                                                            max_iterations=10**8), comm=comm)
    finally:
        comm.close()
    digest = float(np.sum(r.x)) + float(np.sum(r.y))
    allv = [None] * ws
    dist.all_gather_object(allv, (r.iterations, r.restarts, r.objective, digest, tl.status.value,
                                  tl.iterations))
    ok = True
    out = {"world_size": ws}
    if rank == 0:
        same = all(v == allv[0] for v in allv)           # replicated results on every rank
        out.update(ranks_agree=same, iterations=r.iterations, ref_iterations=ref.iterations,
                   restarts=r.restarts, ref_restarts=ref.restarts, objective=r.objective,
                   ref_objective=ref.objective, time_limit_status=tl.status.value,
                   time_limit_iterations=tl.iterations, block_nnz=r.device_stats["block_nnz"])
        ok = (same and r.status.value == ref.status.value == "optimal-tolerance"
              and abs(r.objective - ref.objective) <= 1e-6 * abs(ref.objective)
              and abs(r.iterations - ref.iterations) <= max(32, 0.02 * ref.iterations)
              and tl.status.value == "time-limit")
        out["ok"] = ok
        print(json.dumps(out), flush=True)
    flag = [ok]
    dist.broadcast_object_list(flag, src=0)
    dist.destroy_process_group()
    sys.exit(0 if flag[0] else 1)


if __name__ == "__main__":
    main()
