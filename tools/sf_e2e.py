"""End-to-end successive-fixing wall time (north star "reported results"):
the reference's own transmission-filtered two-stage driver (scuckit.driver.run,
driver.py:203-325) on a synthetic instance, with its LP relaxations either on
the reference CPU HPR solver (--backend cpu) or routed to the B200 engine by
hprlp.install() (--backend gpu; nothing else in the driver changes).

Needs the reference package: baseline/_ref (travels to the GPU box) or
/root/reference/pkg/src.  Prints one JSON line with the driver's RunReport
timings (lp_relaxations / other / total), status, objective and passes.

    python tools/sf_e2e.py --backend gpu --config C1 --time-limit 1500
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "scuckit")):
        sys.path.append(p)
        break

ap = argparse.ArgumentParser()
ap.add_argument("--backend", choices=["gpu", "cpu"], default="gpu")
ap.add_argument("--config", default="C1")
ap.add_argument("--time-limit", type=float, default=1500.0)
ap.add_argument("--out", default=None)
ap.add_argument("--bb", action="store_true", help="install(bb=True): speculative sibling solves")
ap.add_argument("--shutdown-feasible", action="store_true",
                help="cap initial outputs at the shutdown limit (scuc.generate_instance)")
a = ap.parse_args()

from scuckit import driver, parse_instance  # noqa: E402

from paper_2510_10891_b200 import scuc  # noqa: E402

doc = scuc.generate_instance(**scuc.CONFIGS[a.config], shutdown_feasible=a.shutdown_feasible)
inst = parse_instance(doc)
if a.backend == "gpu":
    from paper_2510_10891_b200 import hprlp
    hprlp.install(bb=a.bb)

# wall time of the driver's per-pass model construction (driver.py:210, :249-250)
# and of every LP solve, whichever backend is bound
_timed = {"compute_ptdf_s": [], "build_model_s": [], "lp_solve_s": [], "screen_s": [],
          "violations": [], "model_nnz": []}


def _wrap(mod, name, key):
    fn = getattr(mod, name)

    def timed(*args, **kw):
        t = time.perf_counter()
        try:
            return fn(*args, **kw)
        finally:
            _timed[key].append(time.perf_counter() - t)
    setattr(mod, name, timed)


import scuckit.hprlp  # noqa: E402
_wrap(driver, "compute_ptdf", "compute_ptdf_s")
_wrap(driver, "build_model", "build_model_s")
_wrap(scuckit.hprlp, "solve", "lp_solve_s")
_wrap(driver, "screen_violations", "screen_s")
_bm, _sv = driver.build_model, driver.screen_violations


def _bm_count(*args, **kw):
    out = _bm(*args, **kw)
    _timed["model_nnz"].append(int(out[0].lp.matrix.csr.nnz))
    return out


def _sv_count(*args, **kw):
    out = _sv(*args, **kw)
    _timed["violations"].append(len(out))
    return out


driver.build_model, driver.screen_violations = _bm_count, _sv_count
t0 = time.perf_counter()
try:
    rep = driver.run(inst, driver.DriverConfig(time_limit=a.time_limit))
except Exception as exc:          # e.g. a pass-2 model beyond int32 indexing
    wall = time.perf_counter() - t0
    out = {"backend": a.backend, "config": a.config, "shutdown_feasible": a.shutdown_feasible,
           "time_limit_s": a.time_limit, "wall_s": wall,
           "error": f"{type(exc).__name__}: {exc}", "host_cores": os.cpu_count(),
           **{k: v for k, v in _timed.items() if k != "lp_solve_s"},
           "lp_solves": len(_timed["lp_solve_s"]), "lp_solve_s_total": sum(_timed["lp_solve_s"])}
    print(json.dumps(out), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(json.dumps(out) + "\n")
    sys.exit(0)
wall = time.perf_counter() - t0
d = rep.to_json_dict()
out = {"backend": a.backend, "config": a.config, "shutdown_feasible": a.shutdown_feasible,
       "time_limit_s": a.time_limit,
       "wall_s": wall, "status": d["status"], "exit_code": d["exit_code"],
       "objective": d["objective"], "timings": d["timings"], "nodes_total": d["nodes_total"],
       "fixing": d["fixing"], "passes": d["passes"], "monitored_rows": len(d["monitored"]),
       "host_cores": os.cpu_count(),
       "compute_ptdf_s": _timed["compute_ptdf_s"], "build_model_s": _timed["build_model_s"],
       "screen_s": _timed["screen_s"], "violations": _timed["violations"],
       "model_nnz": _timed["model_nnz"],
       "lp_solves": len(_timed["lp_solve_s"]), "lp_solve_s_total": sum(_timed["lp_solve_s"])}
if a.backend == "gpu":
    from paper_2510_10891_b200 import bb
    out["bb_speculation"] = dict(bb.STATS)
line = json.dumps(out)
print(line, flush=True)
if a.out:
    with open(a.out, "w") as fh:
        fh.write(line + "\n")
