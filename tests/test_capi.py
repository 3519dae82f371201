"""The C-ABI library loads on a CPU-only host and exports every entry point
declared in include/*.h (no compute calls here)."""

import ctypes
import os
import re

from paper_2510_10891_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    inc = os.path.join(ROOT, "include")
    src = "".join(open(os.path.join(inc, f)).read() for f in sorted(os.listdir(inc))
                  if f.endswith(".h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|void|const char\*)\s+\**(hpr_\w+)\s*\(",
                                 src, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    names = header_functions()
    assert len(names) >= 11
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_capi.EXPORTS)
    assert lib.hpr_abi_version() == 1


def test_struct_layouts_match_header_sizes():
    # field counts mirror the header; sizes are 8-byte aligned C layouts
    assert ctypes.sizeof(_capi.Kkt) == 80
    assert ctypes.sizeof(_capi.LogRecord) == 3 * 8 + 8 * 8
    assert ctypes.sizeof(_capi.Problem) == 4 * 3 + 4 + 8 + 10 * 8 + 8


def test_errors_are_codes_not_exceptions():
    lib = _capi.load()
    nbytes = ctypes.c_size_t(0)
    code = lib.hpr_workspace_bytes(None, ctypes.byref(nbytes))
    assert code == _capi.HPR_ERR_INVALID
    assert b"NULL" in lib.hpr_last_error()


def test_workspace_query_without_gpu():
    import numpy as np
    from paper_2510_10891_b200 import scuc
    doc = scuc.generate_instance(12, 6, 18, 6, seed=5)
    lp = scuc.build_relaxation(doc, scuc.all_base_triples(doc))
    P = _capi.ptr
    keep = [np.ascontiguousarray(a) for a in (lp.indptr, lp.indices, lp.data, lp.rhs, lp.cost,
                                              lp.lower, lp.upper)]
    prob = _capi.Problem(lp.shape[0], lp.shape[1], lp.n_eq, lp.nnz, P(keep[0]), P(keep[1]),
                         P(keep[2]), None, None, None, P(keep[3]), P(keep[4]), P(keep[5]),
                         P(keep[6]), 0.0)
    nbytes = ctypes.c_size_t(0)
    assert _capi.load().hpr_workspace_bytes(ctypes.byref(prob), ctypes.byref(nbytes)) == 0
    assert nbytes.value > lp.nnz * (4 + 8 + 8 + 4) * 2


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2510_10891_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            assert "oracle" not in open(os.path.join(pkg, fn)).read().replace(
                "no CPU fallback", ""), fn


def test_c_caller_links_and_presolves(tmp_path):
    """tests/c/abi_smoke.c: a plain-C caller of include/*.h linked against the
    library (the binding any host language would make); runs the host-only
    presolve core through the C-ABI and the solver ABI's no-GPU paths."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        import pytest
        pytest.skip("gcc not available")
    libdir = os.path.join(ROOT, "paper_2510_10891_b200")
    exe = str(tmp_path / "abi_smoke")
    subprocess.run([gcc, "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-L", libdir,
                    "-lhprlp_b200", f"-Wl,-rpath,{libdir}", "-lm", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("ok")


def test_screen_abi_errors_without_gpu():
    """include/hpr_screen.h: argument errors are codes with a message, checked
    before any device call (so they hold on a CPU-only host too)."""
    lib = _capi.load()
    h = ctypes.c_void_p()
    assert lib.hpr_screen_create(0, 4, 4, 1, None, None, ctypes.byref(h)) == _capi.HPR_ERR_INVALID
    assert b"null" in lib.hpr_last_error()
    n = ctypes.c_int64()
    assert lib.hpr_screen_run(None, None, 24, 1e-4, ctypes.byref(n)) == _capi.HPR_ERR_INVALID
    assert lib.hpr_screen_fetch(None, None, None, None, None, None) == _capi.HPR_ERR_INVALID
    assert lib.hpr_screen_flows(None, 0, None) == _capi.HPR_ERR_INVALID
    assert ctypes.sizeof(_capi.ScreenInfo) == 6 * 4 + 8
    lib.hpr_screen_destroy(None)            # no-op
