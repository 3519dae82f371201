"""Where does e2e setup time go?  (Engine creation = host layout + upload;
device setup = scaling + power method + initial check.)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2510_10891_b200 import hprlp, scuc
t = time.perf_counter(); doc, mon, lpa = scuc.build_config("C4"); print("build", round(time.perf_counter() - t, 2))
for rep in range(2):
    lp = lpa.to_lp()
    t = time.perf_counter(); csc = lp.matrix.csc; tc = time.perf_counter() - t
    lp = lpa.to_lp()
    t = time.perf_counter(); eng = hprlp.Engine(lp); torch.cuda.synchronize(); te = time.perf_counter() - t
    t = time.perf_counter()
    x, y, z, st, _ = eng.solve_raw(hprlp.SolverConfig(tolerance=1e-4, ruiz=False, max_iterations=0))
    ts = time.perf_counter() - t
    print(f"scipy tocsc {tc:.2f}s | Engine() {te:.2f}s | solve(max_it=0) {ts:.2f}s (device setup {st.setup_seconds:.3f}s, power its {st.power_iterations})")
    eng.close()
