"""Split of the end-to-end hprlp.solve time at C4 (bench.py e2e): Engine()
(upload + device layout), solve_raw (device setup + loop + copy back).
Usage: time_e2e.py [fp64|fp32]; HPR_VERBOSE=1 adds the per-phase host times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_10891_b200 import hprlp, scuc
doc, mon, lpa = scuc.build_config("C4")
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
cfg = hprlp.SolverConfig(tolerance=1e-4, ruiz=False, max_iterations=200000,
                         precision=hprlp.Precision(prec))
for rep in range(2):
    lp = lpa.to_lp()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = hprlp.Engine(lp)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x, y, z, st, _ = eng.solve_raw(cfg)
    t2 = time.perf_counter()
    print(f"rep {rep}: Engine() {t1 - t0:.3f}s solve_raw {t2 - t1:.3f}s (loop {st.loop_seconds:.3f}s "
          f"device setup {st.setup_seconds:.3f}s) iterations {st.iterations}", flush=True)
    eng.close()
    t0 = time.perf_counter()
    res = hprlp.solve(lpa.to_lp(), cfg)
    print(f"rep {rep}: hprlp.solve wall {time.perf_counter() - t0:.3f}s", flush=True)
