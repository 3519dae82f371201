"""Small-LP regime (B&B node LPs, fixing rounds at C1/C2 size): engine
creation time, it/s and time-to-tolerance through hprlp.solve, per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_10891_b200 import hprlp, scuc  # noqa: E402

for name, tri, tol in (("C1", None, 1e-4), ("C1", None, 1e-6), ("C2", 500, 1e-4)):
    if tri is None:
        doc = scuc.generate_instance(**scuc.CONFIGS[name])
        lpa = scuc.build_relaxation(doc, scuc.all_base_triples(doc))
    else:
        doc, mon, lpa = scuc.build_config(name, n_triples=tri)
    lp = lpa.to_lp()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = hprlp.Engine(lp)
    t_create = time.perf_counter() - t0
    x, y, z, st, _ = eng.solve_raw(hprlp.SolverConfig(tolerance=tol, ruiz=False,
                                                      max_iterations=400000))
    t_solve = time.perf_counter() - t0 - t_create
    eng.close()
    print(json.dumps({"config": name, "triples": tri, "shape": list(lpa.shape), "nnz": int(lpa.nnz),
                      "tol": tol, "create_s": t_create, "solve_s": t_solve,
                      "iterations": int(st.iterations), "loop_s": st.loop_seconds,
                      "it_per_s": st.iterations / max(st.loop_seconds, 1e-9),
                      "us_per_it": 1e6 * st.loop_seconds / max(st.iterations, 1),
                      "status": int(st.status)}), flush=True)
