"""ctypes binding of libhprlp_b200.so (include/hprlp_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make``)
and loaded from this package directory.  There is no fallback: if the
shared object is missing or no CUDA device is present, ``lib()`` raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libhprlp_b200.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)

HPR_OPTIMAL, HPR_ITERATION_LIMIT, HPR_TIME_LIMIT, HPR_NUMERICAL_FAILURE = 0, 1, 2, 3
HPR_FP64, HPR_FP32 = 0, 1
HPR_FLAG_NO_REORDER = 1
HPR_FLAG_NO_FOLD = 2
HPR_FLAG_NO_RUNS = 4
HPR_FLAG_NO_PANELS = 8
HPR_BENCH_IN_ITERATION = 0x100      # hpr_bench_kernel: time the kernel inside its iteration
HPR_ERR_INVALID, HPR_ERR_CUDA, HPR_ERR_NOMEM, HPR_ERR_EMPTY, HPR_ERR_POWER_NULL = -1, -2, -3, -4, -5

EXPORTS = ("hpr_abi_version", "hpr_last_error", "hpr_workspace_bytes", "hpr_create",
           "hpr_destroy", "hpr_solve", "hpr_get_log", "hpr_matvec", "hpr_kkt_residual",
           "hpr_power_method", "hpr_iterate", "hpr_resume", "hpr_bench_kernel",
           "hpr_get_layout", "hpr_nccl_unique_id", "hpr_nccl_comm_init",
           "hpr_nccl_comm_destroy",
           # include/hpr_presolve.h (host-only presolve core)
           "hpr_presolve_run", "hpr_presolve_info", "hpr_presolve_fetch", "hpr_presolve_free",
           "hpr_presolve_reduce",
           # include/hpr_screen.h (device flow screen)
           "hpr_screen_create", "hpr_screen_run", "hpr_screen_fetch", "hpr_screen_flows",
           "hpr_screen_bench", "hpr_screen_info_get", "hpr_screen_destroy",
           "hpr_fp64_peak_bench")

_p = C.c_void_p


class Problem(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("n_eq", C.c_int32), ("nnz", C.c_int64),
                ("indptr", _p), ("indices", _p), ("data", _p),
                ("t_indptr", _p), ("t_indices", _p), ("t_data", _p),
                ("rhs", _p), ("cost", _p), ("lower", _p), ("upper", _p),
                ("offset", C.c_double)]


class Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("stream", _p), ("workspace", _p),
                ("workspace_bytes", C.c_size_t), ("flags", C.c_int32), ("nccl_comm", _p),
                ("world_size", C.c_int32), ("rank", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_iterations", C.c_int64),
                ("time_limit", C.c_double), ("time_elapsed", C.c_double),
                ("precision", C.c_int32), ("has_sigma0", C.c_int32), ("sigma0", C.c_double),
                ("restart_beta", C.c_double), ("restart_stall", C.c_int64),
                ("sigma_damping", C.c_double), ("ruiz", C.c_int32), ("ruiz_iters", C.c_int32),
                ("pock_chambolle", C.c_int32), ("normalize_rhs_objective", C.c_int32),
                ("check_every", C.c_int32), ("power_tol", C.c_double),
                ("power_inflation", C.c_double), ("power_max_iter", C.c_int32),
                ("power_start", _p), ("power_start_count", C.c_int32),
                ("log_residuals", C.c_int32), ("log_every_iteration", C.c_int32)]


class Kkt(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("primal", "box", "dual", "rel_primal", "rel_box",
                                          "rel_dual", "primal_objective", "dual_objective",
                                          "gap", "rel_gap")]


class Stats(C.Structure):
    _fields_ = [("status", C.c_int32), ("precision_used", C.c_int32),
                ("iterations", C.c_int64), ("restarts", C.c_int64),
                ("sigma_final", C.c_double), ("lam", C.c_double), ("objective", C.c_double),
                ("kkt", Kkt), ("n_log", C.c_int64), ("power_iterations", C.c_int32),
                ("power_converged", C.c_int32), ("setup_seconds", C.c_double),
                ("loop_seconds", C.c_double), ("gpu_launches", C.c_int64),
                ("checks", C.c_int64)]


class LogRecord(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("epoch", C.c_int64), ("k", C.c_int64)] + [
        (k, C.c_double) for k in ("rel_primal", "rel_dual", "rel_box", "rel_gap", "sigma",
                                  "primal", "box", "dual")]


class Layout(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("n_eq", C.c_int32),
                ("folded_rows", C.c_int32), ("nnz", C.c_int64), ("folded_nnz", C.c_int64),
                ("tiles_a", C.c_int32), ("tiles_at", C.c_int32), ("tiles_f", C.c_int32),
                ("tiles_ft", C.c_int32), ("reordered", C.c_int32), ("folded", C.c_int32),
                ("workspace_bytes", C.c_size_t), ("panel_cols", C.c_int64),
                ("panel_nnz", C.c_int64), ("f_nnz", C.c_int64), ("ft_nnz", C.c_int64),
                ("index_free_nnz_f", C.c_int64), ("fused", C.c_int32), ("row_panel_groups", C.c_int32)]


class ScreenInfo(C.Structure):
    _fields_ = [("n_lines", C.c_int32), ("n_buses", C.c_int32), ("n_tables", C.c_int32),
                ("bus_pitch", C.c_int32), ("splits", C.c_int32), ("ctas_per_sm", C.c_int32),
                ("table_bytes", C.c_size_t)]


class HprError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libhprlp_b200 error {code}: {msg}")
        self.code = code


_LIB = None


def load(path: str | None = None):
    """Load the shared library and declare signatures (no device needed).
    HPR_LIB overrides the in-tree path (kernel-variant experiments)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = path or os.environ.get("HPR_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (or make) first")
    # torch first: the library's libnccl.so.2 dependency must resolve to the NCCL
    # torch bundles (loading the system NCCL first breaks a later `import torch`)
    import torch  # noqa: F401
    lib = C.CDLL(path)
    lib.hpr_abi_version.restype = C.c_int32
    lib.hpr_last_error.restype = C.c_char_p
    lib.hpr_workspace_bytes.argtypes = [C.POINTER(Problem), C.POINTER(C.c_size_t)]
    lib.hpr_create.argtypes = [C.POINTER(Problem), C.POINTER(Options), C.POINTER(_p)]
    lib.hpr_destroy.argtypes = [_p]
    lib.hpr_destroy.restype = None
    lib.hpr_solve.argtypes = [_p, C.POINTER(Params), _p, _p, _p, _p, _p, _p, C.POINTER(Stats)]
    lib.hpr_get_log.argtypes = [_p, C.POINTER(LogRecord), C.c_int64, C.POINTER(C.c_int64)]
    lib.hpr_matvec.argtypes = [_p, C.c_int32, _p, _p]
    lib.hpr_kkt_residual.argtypes = [_p, _p, _p, _p, C.POINTER(Kkt)]
    lib.hpr_power_method.argtypes = [_p, C.c_double, C.c_int32, C.c_double, _p, C.c_int32,
                                     C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32)]
    lib.hpr_iterate.argtypes = [_p, C.c_int32, C.c_double, C.c_double, C.c_int64] + [_p] * 12
    lib.hpr_resume.argtypes = [_p, C.c_int64, C.c_double, C.POINTER(Stats)]
    lib.hpr_bench_kernel.argtypes = [_p, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
    lib.hpr_get_layout.argtypes = [_p, C.POINTER(Layout)]
    lib.hpr_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8 * 128)]
    lib.hpr_nccl_comm_init.argtypes = [C.POINTER(C.c_uint8 * 128), C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(_p)]
    lib.hpr_nccl_comm_destroy.argtypes = [_p]
    lib.hpr_nccl_comm_destroy.restype = None
    lib.hpr_presolve_run.argtypes = [_p, C.c_int32, C.POINTER(_p)]
    lib.hpr_presolve_info.argtypes = [_p, _p]
    lib.hpr_presolve_fetch.argtypes = [_p] * 8
    lib.hpr_presolve_free.argtypes = [_p]
    lib.hpr_presolve_free.restype = None
    lib.hpr_presolve_reduce.argtypes = [C.c_int32, C.c_int32] + [_p] * 8 + [C.POINTER(C.c_int64)]
    lib.hpr_screen_create.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.POINTER(_p), _p, C.POINTER(_p)]
    lib.hpr_screen_run.argtypes = [_p, _p, C.c_int32, C.c_double, C.POINTER(C.c_int64)]
    lib.hpr_screen_fetch.argtypes = [_p] * 6
    lib.hpr_screen_flows.argtypes = [_p, C.c_int32, _p]
    lib.hpr_screen_bench.argtypes = [_p, C.c_int32, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]
    lib.hpr_screen_info_get.argtypes = [_p, C.POINTER(ScreenInfo)]
    lib.hpr_screen_destroy.argtypes = [_p]
    lib.hpr_screen_destroy.restype = None
    lib.hpr_fp64_peak_bench.argtypes = [C.c_int32, C.POINTER(C.c_double)]
    _LIB = lib
    return lib


def check(code: int):
    if code != 0:
        msg = load().hpr_last_error().decode(errors="replace")
        raise HprError(code, msg)


def ptr(a) -> C.c_void_p | None:
    """Address of a contiguous numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags.c_contiguous
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())
