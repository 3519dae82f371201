"""Flow-screen benchmark at C4 scale (13,659 buses, 20,467 lines, 36 periods;
one base-case PTDF table of 2.24 GB FP64): the device screen
(``screen.screen_violations`` / ``FlowScreen``) against the reference
algorithm on the host (``oracle/screen_oracle.py``: ``table @ inj`` in
numpy/OpenBLAS with every host thread, then the reference's Python loop).

    python tools/screen_bench.py [--buses 13659 --gens 4092 --lines 20467 --periods 36]

Prints one JSON line: product / epilogue device times (CUDA events over
``reps`` relaunches, inputs resident), the algorithmic bytes and flops per
launch, HBM and FP64 roofline fractions, end-to-end time through the public
call (host point in, sorted Violation list out) and the CPU baseline."""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import screen_oracle  # noqa: E402  (CPU baseline leg only)
from paper_2510_10891_b200 import scuc, screen  # noqa: E402

HBM_GBS = 6548.2
FP64_TFLOPS_NOMINAL = 37.0   # B200 datasheet FP64 (= FP64 tensor); no measured figure in MEASURED_PEAKS


def full_ptdf(doc, device):
    """All rows of the base PTDF via scuc._ptdf_rows_direct (torch LU on the GPU)."""
    inst = scuc.Instance(doc)
    net = inst.net
    return scuc._ptdf_rows_direct(net.n_b, net.fb, net.tb, net.react, net.ref,
                                  list(range(len(net.fb))), device=device)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--buses", type=int, default=13659)
    ap.add_argument("--gens", type=int, default=4092)
    ap.add_argument("--lines", type=int, default=20467)
    ap.add_argument("--periods", type=int, default=36)
    ap.add_argument("--seed", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cpu", type=int, default=1, help="time the host reference leg")
    a = ap.parse_args()
    t0 = time.perf_counter()
    doc = scuc.generate_instance(a.buses, a.gens, a.lines, a.periods, seed=a.seed)
    tab = full_ptdf(doc, "cuda")
    t_build = time.perf_counter() - t0
    inst = screen.instance_view(doc)
    ptdf = screen.Tables({"base": tab})

    # a dispatch that loads the network: every unit on at 80-100% of p_max
    from paper_2510_10891_b200 import screen as S
    u, pp, pen, n_cols = S.column_blocks(inst)
    rng = np.random.default_rng(a.seed)
    x = np.zeros(n_cols)
    x[u] = 1.0
    span = np.array([[g["p_max"] - g["p_min"]] for g in doc["generators"]])
    x[pp] = span * rng.uniform(0.8, 1.0, size=u.shape)

    t1 = time.perf_counter()
    v_first = screen.screen_violations(x, inst, ptdf)          # uploads the table
    t_first = time.perf_counter() - t1
    e2e = []
    for _ in range(5):
        t1 = time.perf_counter()
        v = screen.screen_violations(x, inst, ptdf)
        e2e.append(time.perf_counter() - t1)
    scr = screen.screen_for(ptdf, inst)
    us_prod, us_epi = scr.bench(a.reps)
    info = scr.info()
    L, B, T = a.lines, a.buses, a.periods
    tp = -(-T // 8) * 8
    bytes_prod = L * B * 8 + B * T * 8 + info["splits"] * L * tp * 8
    flops = 2.0 * L * B * T
    gbs = bytes_prod / us_prod / 1e3
    tfl = flops / us_prod / 1e6
    out = {
        "workload": f"flow screen: {B} buses x {L} lines x {T} periods, base-case PTDF (FP64)",
        "violations": len(v), "first_call_s": t_first, "build_s": t_build,
        "e2e_s": float(np.median(e2e)),
        "product_us": us_prod, "epilogue_us": us_epi,
        "bytes_per_launch": bytes_prod, "flops_per_launch": flops,
        "achieved_gbs": gbs, "hbm_frac": gbs / HBM_GBS,
        "achieved_tflops": tfl, "fp64_frac_nominal": tfl / FP64_TFLOPS_NOMINAL,
        "bound": "fp64" if flops / FP64_TFLOPS_NOMINAL / 1e12 > bytes_prod / HBM_GBS / 1e9 else "hbm",
        "info": info, "same_as_first": [w.triple for w in v] == [w.triple for w in v_first],
    }
    if a.cpu:
        inj = S.injections(x, inst)
        t1 = time.perf_counter()
        flows = tab @ inj
        out["cpu_gemm_s"] = time.perf_counter() - t1
        t1 = time.perf_counter()
        ref = screen_oracle.screen([tab], [[ln.limit for ln in inst.lines]], ["base"],
                                   [ln.lid for ln in inst.lines], inj, (), 1e-4)
        out["cpu_screen_s"] = time.perf_counter() - t1
        out["cpu_threads"] = os.cpu_count()
        out["cpu_same_triple_set"] = {r[:3] for r in ref} == {w.triple for w in v}
        out["max_flow_diff"] = float(np.abs(scr.flows(0) - flows).max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
