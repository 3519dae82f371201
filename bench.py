#!/usr/bin/env python
"""HPR-LP benchmark on the synthetic 13,659-bus SCUC LP relaxation.

Workload (BASELINE.json configs[3], SURVEY.md §8(d) "C4"): 13,659 buses,
4,092 units, 20,467 lines, 36 periods, 1,000 seeded base-case flow triples;
the LP relaxation of the SCUC MILP (1.77M rows x 1.67M cols, ~44M nnz)
built by paper_2510_10891_b200.scuc (random-init data, no datasets).

A *step* is one HPR check block: 16 fused iterations + the master-space
KKT check / restart controller (hprlp.py:393-446), device-resident.
`value` = HPR iterations/s over K steps (CUDA events on the engine stream,
max over ranks).  `e2e` = the same metric through the public API
(hprlp.solve from host numpy arrays: upload, setup, solve to 1e-4, copy
back).  The matrix stream (>1 GB per iteration) exceeds L2, so no flush is
needed between steps.

    python bench.py [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N     (independent replicas)
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HPR iterations/s (time-to-1e-4 KKT in e2e) on 13659-bus SCUC LP"
BLOCK = 16


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--triples", type=int, default=None)
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--e2e-max-iter", type=int, default=200_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-screen", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--mode", default="replicas", choices=["replicas", "partitioned"],
                    help="N>1: independent replicas (weak scaling) or one LP row-partitioned "
                         "over the N GPUs with NCCL (strong scaling)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 5 ms during
    the timed region through NVML (the same counters nvidia-smi reports);
    falls back to nvidia-smi polling when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.active = [], [], set()
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while True:
            self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
            self.mx.append(float(mx))
            bits = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            for name, attr in self.REASONS:
                if bits & getattr(N, attr):
                    self.active.add(name)
            if self._stop.wait(0.005):
                break
        N.nvmlShutdown()

    def _smi(self):
        while True:
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                r = [v.strip() for v in out.split(",")]
                self.sm.append(float(r[0]))
                self.mx.append(float(r[1]))
                for k, (name, _) in enumerate(self.REASONS):
                    if r[2 + k].lower() == "active":
                        self.active.add(name)
            except Exception:
                pass
            if self._stop.wait(0.2):
                break

    def _run(self):
        try:
            self._nvml()
        except Exception:
            self._smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.active), "samples": len(self.sm)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel_key, config):
    """Per-launch DRAM bytes of the dominant kernel on this config from the
    committed ncu capture summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(config, {}).get(kernel_key)
    except Exception:
        return None


def workload(args):
    """The config's description (scuc.CONFIGS; C4 + 1000 base triples is the
    BASELINE.json headline)."""
    from paper_2510_10891_b200 import scuc
    c = scuc.CONFIGS[args.config]
    n = args.triples or {"C1": -1, "C2": 500, "C3": 2000, "C4": 1000, "C5": 20000}[args.config]
    kind = (f"N-1 flow triples over {c['n_contingencies']} line outages"
            if args.config == "C5" else "base flow triples")
    tri = "all base flow triples" if n < 0 else f"{n} sampled {kind}"
    return (f"{args.config}: synthetic {c['n_buses']}-bus/{c['n_gens']}-unit/{c['n_periods']}-period "
            f"SCUC LP relaxation + {tri}")


def config_dict(args, m, n, nnz, ws, partitioned):
    """The `config` object both arms print (identical, so the driver's
    same-config check holds); per-arm details live outside it."""
    return {"workload": workload(args), "rows": int(m), "cols": int(n), "nnz": int(nnz),
            "l2": "inputs larger than L2 (matrix stream > 1 GB/iteration)",
            "parallelism": (f"rowpart{ws}" if partitioned else
                            (f"replicas{ws}" if ws > 1 else "single"))}


def build_lp(args, device):
    from paper_2510_10891_b200 import scuc
    t = time.perf_counter()
    doc, mon, lpa = scuc.build_config(args.config, n_triples=args.triples)
    return lpa, time.perf_counter() - t, doc


def bytes_model(m, n, nnz, s):
    """Algorithmic HBM bytes per launch of each kernel of
    one iteration, and B_iter = core + check/16 for the whole iteration
    (the survey's fused-iteration figure; the engine's extra product-vector
    round trip is not counted as useful work)."""
    spmv_a = nnz * (s + 4) + 4 * (m + 1) + s * n + s * m              # A x~: stream, gather, write
    spmv_at = nnz * (s + 4) + 4 * (n + 1) + s * m + s * n             # A^T y
    upd_primal = s * 11 * n                                           # 8 reads + 3 writes per column
    upd_dual = s * 5 * m                                              # 4 reads + 1 write per row
    core = 2 * nnz * (s + 4) + 4 * (m + n + 2) + s * (11 * n + 5 * m)
    chk = 2 * nnz * 12 + 4 * (m + n + 2) + 8 * (8 * n + 4 * m) + 8 * (2 * n + m)
    return {"spmv_A": spmv_a, "spmv_AT": spmv_at, "update_primal": upd_primal,
            "update_dual": upd_dual, "core": core, "check": chk, "iter": core + chk / BLOCK}


def cpu_baseline_sample(lpa, lam, sigma, precision):
    """The oracle (numpy/scipy restatement of the reference, single-threaded
    SpMV) timed on one HPR block of the same LP: 16 iterations + 1 check,
    after its own scaling (setup excluded; lambda/sigma from the GPU run)."""
    from oracle import hpr_oracle as O
    cfg = O.OracleConfig(tolerance=1e-4, ruiz=False, precision=precision)
    p = O.Problem.from_lp(lpa)
    sc = O.Scaling(p, cfg)
    w = sc.work
    dt = cfg.dtype
    if dt == np.float32:
        w = O.Problem(w.a.cast(np.float32), w.rhs.astype(dt), w.cost.astype(dt),
                      w.lower.astype(dt), w.upper.astype(dt), w.n_eq)
    m, n = p.a.shape
    st = O.HprIterate(O.box(np.zeros(n), sc.work.lower, sc.work.upper), np.zeros(m), np.zeros(n),
                      sigma, lam, dt)
    t0 = time.perf_counter()
    for _ in range(BLOCK):
        st.step(w)
    O.kkt(p, *sc.to_master(st.bx, st.by, st.bz))
    el = time.perf_counter() - t0
    return BLOCK / el, el


FP64_TFLOPS_NOMINAL = 37.0   # B200 datasheet FP64 / FP64 tensor; MEASURED_PEAKS has no FP64 figure


def screen_leg(doc, x, reps):
    """The post-MILP flow screen (driver.screen_violations, driver.py:165-200;
    SURVEY 8(f) rank 3) on the config's base-case PTDF at the e2e LP point:
    device product/epilogue times (CUDA events, inputs resident), the public
    call end to end (host point in, sorted Violation list out), and the host
    BLAS product the reference runs (driver.py:186) timed beside it."""
    import numpy as np
    from paper_2510_10891_b200 import scuc, screen
    t0 = time.perf_counter()
    net = scuc.Instance(doc).net
    tab = scuc._ptdf_rows_direct(net.n_b, net.fb, net.tb, net.react, net.ref,
                                 list(range(len(net.fb))), device="cuda")
    t_ptdf = time.perf_counter() - t0
    inst = screen.instance_view(doc)
    ptdf = screen.Tables({"base": tab})
    t0 = time.perf_counter()
    first = screen.screen_violations(x, inst, ptdf)          # uploads the table once
    t_first = time.perf_counter() - t0
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        v = screen.screen_violations(x, inst, ptdf)
        walls.append(time.perf_counter() - t0)
    scr = screen.screen_for(ptdf, inst)
    us_p, us_e = scr.bench(reps)
    info = scr.info()
    n_l, n_b = tab.shape
    n_t = doc["time_periods"]
    tp = -(-n_t // 8) * 8
    nbytes = n_l * n_b * 8 + n_b * tp * 8 + info["splits"] * n_l * tp * 8
    flops = 2.0 * n_l * n_b * n_t
    inj = screen.injections(x, inst)
    t0 = time.perf_counter()
    _ = tab @ inj
    gemm_s = time.perf_counter() - t0
    from oracle import screen_oracle       # CPU baseline leg only
    t0 = time.perf_counter()
    ref = screen_oracle.screen([tab], [[ln.limit for ln in inst.lines]], ["base"],
                               [ln.lid for ln in inst.lines], inj, (), 1e-4)
    cpu_s = time.perf_counter() - t0
    set_diff = len({r[:3] for r in ref} ^ {w.triple for w in v})
    scr.close()
    tfl = flops / us_p / 1e6
    try:
        peak, peak_kind = screen.fp64_peak_tflops(), "measured (register-only DMMA chains)"
    except Exception:
        peak, peak_kind = FP64_TFLOPS_NOMINAL, "datasheet"
    return {"workload": f"base-case screen: {n_l} lines x {n_b} buses x {n_t} periods "
                        f"(FP64 PTDF {n_l * n_b * 8 / 1e9:.2f} GB resident), e2e LP point",
            "violations": len(v), "same_as_first": [w.triple for w in v] == [w.triple for w in first],
            "product_us": us_p, "epilogue_us": us_e, "splits": info["splits"],
            "roofline": {"bound": "fp64", "achieved": tfl, "peak": peak,
                         "unit": "TFLOP/s", "frac": tfl / peak, "peak_kind": peak_kind,
                         "datasheet_peak": FP64_TFLOPS_NOMINAL, "hbm_gbs": nbytes / us_p / 1e3,
                         "hbm_frac": nbytes / us_p / 1e3 / measured_peak_hbm()[0],
                         "bytes_per_launch": nbytes, "flops_per_launch": flops},
            "e2e_s": float(np.median(walls)), "first_call_s": t_first, "ptdf_build_s": t_ptdf,
            "oracle_set_diff": set_diff,        # triples in one list but not the other
            "cpu_baseline": {"value": cpu_s, "unit": "s", "cores": os.cpu_count(),
                             "kind": "port", "gemm_only_s": gemm_s,
                             "sample": "oracle/screen_oracle.py on the same point: numpy "
                                       "table @ injections with host BLAS (all cores), then the "
                                       "reference's per-(line, period) loop and sort (one core)"}}


def run_b200(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_10891_b200 import hprlp
    from paper_2510_10891_b200.lp import Precision

    lpa, t_build, doc = build_lp(args, f"cuda:{local}")
    m, n = lpa.shape
    nnz = lpa.nnz
    s = 8 if args.precision == "fp64" else 4
    lp = lpa.to_lp()
    partitioned = args.mode == "partitioned"
    cfg = hprlp.SolverConfig(tolerance=1e-4, ruiz=False, precision=Precision(args.precision),
                             max_iterations=max(1, args.warmup) * BLOCK)
    comm = blk = None
    if partitioned:
        from paper_2510_10891_b200 import partition
        if ws == 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            dist.init_process_group("gloo", rank=0, world_size=1)
        comm = hprlp.NcclComm()
        blk = partition.partition_rows(lpa.indptr, lpa.indices, lpa.data, lpa.n_eq, n,
                                       comm.world_size)[comm.rank]
        eng = hprlp.Engine(partition.block_lp(lp, blk), device=local, comm=comm)
        x, y, z, st0, _ = eng.solve_raw(cfg, rows=blk.rows, m_total=m)
    else:
        eng = hprlp.Engine(lp, device=local)
        x, y, z, st0, _ = eng.solve_raw(cfg)              # setup + W warm-up blocks
    lay = eng.layout()
    # timed region: exactly K blocks of the device-resident loop
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        torch.cuda.nvtx.range_push("timed")       # ncu --nvtx-include "timed/" (launch list)
        st = eng.resume(args.steps * BLOCK, tolerance=1e-300)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        # per-kernel times: back-to-back launches between two CUDA events on the
        # engine stream (the launch latency hidden as in the loop's graph)
        names = (("spmv_A", 0), ("spmv_AT", 1), ("update_primal", 2), ("update_dual", 3))
        split = {name: eng.bench_kernel(which, args.kernel_reps) for name, which in names}
        fused = bool(lay.get("fused"))
        # the kernels the loop actually runs: the fused iteration has two
        loop_names = (("spmv_AT+primal", 5), ("spmv_A+dual", 6)) if fused else names
        ktimes = ({name: eng.bench_kernel(which, args.kernel_reps) for name, which in loop_names}
                  if fused else dict(split))
        # upper bounds: events around every launch, each launch followed by the rest
        # of its iteration (the loop's cache state, but each interval also holds
        # the launch ramp that the back-to-back form and the graph hide)
        k_in_iter = {name: eng.bench_kernel(which, args.kernel_reps, in_iteration=True)
                     for name, which in loop_names}
        t_check = eng.bench_kernel(4, 4)     # one KKT check block (mutates state: last)
    if ws > 1:
        torch.distributed.barrier()
    t_loop = st.loop_seconds
    its = int(st.iterations)
    if ws > 1:
        tt = torch.tensor([t_loop], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_loop = float(tt.item())
    value = (1 if partitioned else ws) * its / t_loop

    bm = bytes_model(m, n, nnz, s)
    nf, nnzf = lay["folded_rows"], lay["folded_nnz"]
    # bytes each kernel must move in the engine's own layout (folded twins,
    # index-free chunks, flow panels read from F inside the primal update)
    fz = lay["f_nnz"]
    stored = {"spmv_A": fz * s + 4 * (fz - lay["index_free_nnz_f"]) + 4 * (nf + 1)
                        + s * n + s * nf,
              "spmv_AT": lay["ft_nnz"] * (s + 4) + s * lay["panel_nnz"] + 8 * lay["panel_cols"]
                         + 4 * (n + 1) + s * nf + s * n,
              "update_primal": s * 8 * n,       # z's Halpern update is skipped (never read)
              "update_dual": s * (4 * m + 2 * nf)}
    # fused: the product vector is neither written by the SpMV nor read by the update
    stored["spmv_AT+primal"] = stored["spmv_AT"] + stored["update_primal"] - 2 * s * n
    stored["spmv_A+dual"] = stored["spmv_A"] + stored["update_dual"] - 2 * s * nf
    bm["spmv_AT+primal"] = bm["spmv_AT"] + bm["update_primal"]
    bm["spmv_A+dual"] = bm["spmv_A"] + bm["update_dual"]
    peak, peak_kind = measured_peak_hbm()
    dom = max(ktimes, key=ktimes.get)
    dom_t, dom_b = ktimes[dom], stored[dom]
    ach = dom_b / dom_t / 1e9
    traffic = ncu_traffic(f"{dom}_{args.precision}", args.config)
    it_gbs = bm["iter"] * its / t_loop / 1e9

    out = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_loop / args.steps,
        "higher_is_better": True, "scaling": "strong" if partitioned else "weak",
        "vs_baseline": None,
        "dtype": "f64" if args.precision == "fp64" else "f32", "data": "synthetic",
        "config": config_dict(args, m, n, nnz, ws, partitioned),
        "step": "16 HPR iterations + KKT check",
        "device_layout": {"folded_rows": lay["folded_rows"],
                          "folded_nnz": lay["folded_nnz"],
                          "f_nnz": lay["f_nnz"], "ft_nnz": lay["ft_nnz"],
                          "panel_nnz": lay["panel_nnz"],
                          "index_free_nnz_f": lay["index_free_nnz_f"],
                          "reordered": bool(lay["reordered"]),
                          "twin_folded": bool(lay["folded"])},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak,
                     "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                     "bytes_per_launch": dom_b, "seconds_per_launch": dom_t,
                     "bytes_basis": "algorithmic bytes of the engine's layout (twin rows "
                                    "stored once, index-free flow chunks, A^T y flow panels "
                                    "read from F's rows); CSR-equivalent figure in "
                                    "iteration_roofline (SURVEY 8(d))",
                     "csr_equivalent_bytes_per_launch": bm.get(dom),
                     "peak_kind": peak_kind},
        "iteration_roofline": {"basis": "CSR-equivalent B_iter (SURVEY 8(d))",
                               "bytes_per_iteration": bm["iter"], "achieved_gbs": it_gbs,
                               "frac": it_gbs / peak},
        "kernels": {k: {"us": 1e6 * t, "bytes": stored[k], "gbs": stored[k] / t / 1e9,
                        "frac": stored[k] / t / 1e9 / peak}
                    for k, t in ktimes.items()},
        "kernels_split": ({k: {"us": 1e6 * t, "bytes": stored[k],
                               "frac": stored[k] / t / 1e9 / peak}
                           for k, t in split.items()} if fused else None),
        "iteration_kernels": "fused (updates as SpMV epilogues)" if fused else "split",
        "kernel_timing": "back-to-back launches of each kernel between two CUDA events on "
                         "the engine stream (hpr_bench_kernel)",
        "kernels_in_iteration_us": {k: 1e6 * t for k, t in k_in_iter.items()},
        "iteration_us": 1e6 * t_loop / its,
        "kernel_sum_us": 1e6 * sum(ktimes.values()),
        "check_block_us": 1e6 * t_check,
        "launch_gap_us_per_iteration": 1e6 * (t_loop / its - sum(ktimes.values())
                                              - t_check / BLOCK),
        "gpu_launches": int(st.gpu_launches),
        "setup": {"build_lp_s": t_build, "warmup_setup_s": st0.setup_seconds},
    }
    out["clocks"] = clk.summary()

    if partitioned:
        out["block"] = {"rows": int(blk.rows.size), "nnz": int(blk.nnz)}
    x_point = np.zeros(n)
    if not args.no_e2e and not partitioned:
        # public API from host buffers: upload + setup + solve to 1e-4 + copy back.
        # The benchmark engine is released first, so its 5.6 GB workspace returns
        # to torch's caching allocator and the e2e engine is not charged for a
        # second cudaMalloc the benchmark alone made necessary.
        eng.close()
        del eng
        import gc
        gc.collect()
        lp_host = lpa.to_lp()
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        res = hprlp.solve(lp_host, hprlp.SolverConfig(
            tolerance=1e-4, ruiz=False, precision=Precision(args.precision),
            max_iterations=args.e2e_max_iter))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        job_iters, job_wall = res.iterations, wall
        x_point = res.x                  # the screen leg screens the solved relaxation
        if ws > 1:
            # whole job: every replica solves its own LP; iterations summed, slowest wall
            ti = torch.tensor([float(res.iterations)], device="cuda", dtype=torch.float64)
            tw = torch.tensor([wall], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(ti, op=torch.distributed.ReduceOp.SUM)
            torch.distributed.all_reduce(tw, op=torch.distributed.ReduceOp.MAX)
            job_iters, job_wall = float(ti.item()), float(tw.item())
        h2d = 4 * (m + 1) + 12 * nnz + 8 * (m + 3 * n)     # CSR + rhs/cost/lower/upper
        out["e2e"] = {"value": job_iters / job_wall, "unit": "iterations/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * (2 * n + m),
                      "time_to_tol_s": wall, "status": res.status.value,
                      "iterations": res.iterations, "restarts": res.restarts,
                      "objective": res.objective, "rel_kkt": res.kkt.max_rel,
                      "loop_seconds": res.device_stats.get("loop_seconds"),
                      "device_setup_seconds": res.device_stats.get("setup_seconds"),
                      "engine_create_seconds": res.device_stats.get("create_seconds")}
        if args.precision == "fp64":
            # the paper's setting (FP32 work precision, FP64 master check), same API
            del res, lp_host
            gc.collect()
            lp32 = lpa.to_lp()           # host LP objects are the caller's, built outside the clock
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r32 = hprlp.solve(lp32, hprlp.SolverConfig(
                tolerance=1e-4, ruiz=False, precision=Precision("fp32"),
                max_iterations=args.e2e_max_iter))
            torch.cuda.synchronize()
            w32 = time.perf_counter() - t0
            out["e2e_fp32"] = {"time_to_tol_s": w32, "iterations": r32.iterations,
                               "iterations_per_s": r32.iterations / w32,
                               "status": r32.status.value, "objective": r32.objective,
                               "rel_kkt": r32.kkt.max_rel,
                               "loop_seconds": r32.device_stats.get("loop_seconds"),
                               "engine_create_seconds": r32.device_stats.get("create_seconds"),
                               "fp64_fallback": bool(getattr(r32, "fp64_fallback", False))}
    if rank == 0 and not args.no_screen:
        try:
            out["screen"] = screen_leg(doc, x_point, args.kernel_reps)
        except Exception as exc:          # recorded, never silently replaced
            out["screen"] = {"error": f"{type(exc).__name__}: {exc}"}
    if rank == 0 and not args.no_cpu_baseline:
        v, el = cpu_baseline_sample(lpa, st0.lam, st.sigma_final, args.precision)
        out["cpu_baseline"] = {"value": v, "unit": "iterations/s", "cores": 1, "kind": "port",
                               "sample": f"oracle: {BLOCK} HPR iterations + 1 KKT check on the "
                                         f"same LP ({el:.1f} s; scipy SpMV single-threaded; "
                                         f"{os.cpu_count()} host cores available)"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if comm is not None:
        eng.close()
        comm.close()
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


def run_reference(args):
    """The reference algorithm on the host cores (oracle port — the reference
    package itself is not on the GPU box): one step = one HPR iteration, a
    KKT check every 16th step, on the same LP as the GPU arm."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import hpr_oracle as O
    lpa, t_build, _ = build_lp(args, "cuda:0" if _has_cuda() else None)
    cfg = O.OracleConfig(tolerance=1e-4, ruiz=False, precision=args.precision)
    p = O.Problem.from_lp(lpa)
    t0 = time.perf_counter()
    sc, w, lam, sigma = O.setup(p, cfg)
    t_setup = time.perf_counter() - t0
    m, n = p.a.shape
    st = O.HprIterate(O.box(np.zeros(n), sc.work.lower, sc.work.upper), np.zeros(m), np.zeros(n),
                      sigma, lam, cfg.dtype)

    def step():
        st.step(w)
        if st.total % BLOCK == 0:
            O.kkt(p, *sc.to_master(st.bx, st.by, st.bz))

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    v = args.steps / el
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iterations/s",
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
           "data": "synthetic",
           "config": config_dict(args, m, n, lpa.nnz, ws, args.mode == "partitioned"),
           "step": "1 HPR iteration (KKT check every 16th)",
           "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": 1, "kind": "port",
                            "sample": f"{args.steps} iterations after {args.warmup} warm-up "
                                      f"(oracle setup {t_setup:.1f} s untimed; scipy SpMV "
                                      f"single-threaded, {os.cpu_count()} cores available)"},
           "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)
