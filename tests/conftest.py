import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def reference_available() -> bool:
    """True in the build container where the read-only reference exists
    (never on the GPU box)."""
    if not os.path.isdir(REF_SRC):
        return False
    if REF_SRC not in sys.path:
        sys.path.append(REF_SRC)
    try:
        import scuckit  # noqa: F401
        return True
    except Exception:
        return False


needs_reference = pytest.mark.skipif(not reference_available(),
                                     reason="reference package not present (GPU box)")
