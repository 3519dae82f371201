"""Multi-rank (row-partitioned) HPR path, exercised on CPU with gloo.

The partition planner (product code) and the partitioned algorithm
(oracle/hpr_partitioned.py, the restatement the NCCL engine mode follows)
run with world_size 2; the result must match the single-process oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_10891_b200 import partition, scuc


def _lp():
    doc = scuc.generate_instance(30, 12, 45, 8, seed=3)
    return scuc.build_relaxation(doc, scuc.sample_monitored(doc, 60, 3))


def _twin_lp(seed=0):
    """A random bounded-feasible LP (the golden-fixture recipe) extended with
    range constraints lo <= a.x <= hi written as the (a, -a) twin rows the
    SCUC flow limits produce; small enough for a fast gloo solve."""
    import scipy.sparse as sp
    from tests.golden_io import FixtureLp
    rng = np.random.default_rng(seed)
    n, m0, k = 24, 14, 6
    a = rng.standard_normal((m0, n)) * (rng.uniform(size=(m0, n)) < 0.4)
    a[np.arange(m0), rng.integers(0, n, m0)] += 1.0
    lower, upper = -rng.uniform(1, 3, n), rng.uniform(1, 3, n)
    xf = rng.uniform(-0.5, 0.5, n)
    n_eq = 4
    rhs = a @ xf
    rhs[n_eq:] -= rng.uniform(0, 1, m0 - n_eq)
    tw = rng.standard_normal((k, n)) * (rng.uniform(size=(k, n)) < 0.6)
    mid = tw @ xf
    rows = [a] + [np.vstack([tw[i], -tw[i]]) for i in range(k)]
    rhs = np.concatenate([rhs] + [[mid[i] - 0.5, -(mid[i] + 0.5)] for i in range(k)])
    A = sp.csr_matrix(np.vstack(rows))
    A.sort_indices()
    cost = rng.standard_normal(n)
    return FixtureLp(A.indptr, A.indices, A.data, A.shape, rhs, cost, lower, upper, n_eq)


class _Arrays:
    """partition_rows wants CSR arrays; adapt a FixtureLp."""

    def __init__(self, lp):
        c = lp.matrix.csr
        self.indptr, self.indices, self.data = c.indptr, c.indices, c.data
        self.n_eq, self.shape = lp.n_eq, c.shape


def test_partition_covers_balances_and_keeps_twins():
    lpa = _lp()
    for ws in (1, 2, 3, 4):
        blocks = partition.partition_rows(lpa.indptr, lpa.indices, lpa.data, lpa.n_eq,
                                          lpa.shape[1], ws)
        rows = np.concatenate([b.rows for b in blocks])
        assert np.array_equal(np.sort(rows), np.arange(lpa.shape[0]))
        for b in blocks:
            assert np.all(b.rows[:b.n_eq] < lpa.n_eq) and np.all(b.rows[b.n_eq:] >= lpa.n_eq)
            # twin (flow lo, hi) pairs never straddle ranks
            lows = set(b.rows.tolist())
        tot = sum(b.nnz for b in blocks)
        assert max(b.nnz for b in blocks) <= tot / ws + 2 * np.diff(lpa.indptr).max()
        owner = np.empty(lpa.shape[0], int)
        for b in blocks:
            owner[b.rows] = b.rank
        m0 = lpa.shape[0] - 2 * 60
        assert all(owner[i] == owner[i + 1] for i in range(m0, lpa.shape[0], 2))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, cfg_kw, seed, q):
    import torch.distributed as dist
    from oracle import hpr_partitioned as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        lp = _twin_lp(seed)
        arr = _Arrays(lp)
        blocks = partition.partition_rows(arr.indptr, arr.indices, arr.data, arr.n_eq,
                                          arr.shape[1], ws)
        blk = blocks[rank]
        res = P.solve(P.block_from_lp(lp, blk), blk.rows, arr.shape[0], cfg_kw)
        q.put((rank, blk.rows, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_kw,seed", [(dict(tolerance=1e-7, ruiz=False), 0),
                                         (dict(tolerance=1e-7, ruiz=True), 1)])
def test_two_rank_gloo_matches_single_process(cfg_kw, seed):
    from oracle import hpr_oracle as O
    lp = _twin_lp(seed)
    ref = O.solve(lp, O.OracleConfig(**cfg_kw))
    assert ref.status == "optimal-tolerance"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg_kw, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    (r0, rows0, a), (r1, rows1, b) = out
    # replicated state agrees bit for bit across ranks
    assert np.array_equal(a["x"], b["x"]) and a["iterations"] == b["iterations"]
    assert a["status"] == b["status"] == ref.status
    assert a["lam"] == pytest.approx(ref.lam, rel=1e-10)
    assert abs(a["objective"] - ref.objective) <= 1e-6 * max(1.0, abs(ref.objective))
    assert abs(a["iterations"] - ref.iterations) <= max(64, 0.05 * ref.iterations)
    assert len(rows0) > 0 and len(rows1) > 0
    y = np.empty(lp.n_rows)
    y[rows0], y[rows1] = a["y"], b["y"]
    assert O.kkt(O.Problem.from_lp(lp), a["x"], y, a["z"]).max_rel <= cfg_kw["tolerance"] * 1.001


@pytest.mark.gpu
def test_partitioned_engine_multi_rank_cuda():
    """The CUDA partitioned engine (libhprlp_b200.so, NCCL inside the block
    graph) on >= 2 ranks / GPUs, launched by torchrun: the partitioned solve
    matches the single-GPU solve and every rank returns the same result
    (tools/partitioned_check.py).  Skipped on a one-GPU box; the driver's
    multi-GPU run executes it."""
    import subprocess
    import sys
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip(f"needs >= 2 GPUs (this box has {n})")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone",
                          "--local-addr", "127.0.0.1", f"--nproc-per-node={min(n, 4)}",
                          os.path.join(root, "tools", "partitioned_check.py")],
                         capture_output=True, text=True, timeout=1200, cwd=root)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
