"""Host-side LP containers mirroring ``scuckit.lp_kernel`` (plumbing only).

The HPR engine accepts any object shaped like the reference's
``StandardFormLp`` (``scuckit/lp_kernel.py:178-241``): ``.matrix.csr`` (a
canonical scipy CSR, float64), optionally ``.matrix.csc``, and the vectors
``rhs``, ``cost``, ``lower``, ``upper`` plus ``n_eq`` and ``offset``.  When
the reference package is importable its own classes are used unchanged; these
mirrors exist so the engine, its tests and the bench run on a machine where
the reference is absent (the GPU box).  No arithmetic of the solve path lives
here.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np


class Precision(enum.Enum):
    """Mirror of ``lp_kernel.Precision`` (``lp_kernel.py:18-31``)."""

    FP32 = "fp32"
    FP64 = "fp64"

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float32 if self is Precision.FP32 else np.float64)


class SparseMatrix:
    """Canonical CSR + CSC pair (``lp_kernel.py:44-62``)."""

    def __init__(self, matrix, dtype=np.float64):
        import scipy.sparse as sp
        csr = sp.csr_matrix(matrix, dtype=dtype)
        csr.sum_duplicates()
        csr.eliminate_zeros()
        csr.sort_indices()
        self.csr = csr
        self._csc = None
        self.shape = csr.shape
        self.dtype = csr.dtype

    @classmethod
    def from_csr_arrays(cls, indptr, indices, data, shape):
        import scipy.sparse as sp
        return cls(sp.csr_matrix((data, indices, indptr), shape=shape))

    @property
    def csc(self):
        if self._csc is None:
            self._csc = self.csr.tocsc()
            self._csc.sort_indices()
        return self._csc

    @property
    def nnz(self) -> int:
        return self.csr.nnz


@dataclass
class StandardFormLp:
    """min cost.x + offset  s.t.  A x (= first n_eq | >= rest) rhs,
    lower <= x <= upper  (``lp_kernel.py:178-213``)."""

    matrix: SparseMatrix
    rhs: np.ndarray
    cost: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    n_eq: int = 0
    offset: float = 0.0
    row_tags: list = field(default_factory=list)
    col_tags: list = field(default_factory=list)

    @property
    def n_rows(self) -> int:
        return self.matrix.shape[0]

    @property
    def n_cols(self) -> int:
        return self.matrix.shape[1]

    def objective(self, x: np.ndarray) -> float:
        return float(np.dot(np.asarray(self.cost, np.float64),
                            np.asarray(x, np.float64))) + self.offset


class MilpModel:
    """Mirror of ``formulation.MilpModel`` (``formulation.py:100-145``): the
    LP plus integrality marks (what presolve reads and returns)."""

    def __init__(self, lp: StandardFormLp, integrality, vmap=None):
        self.lp = lp
        self.integrality = np.asarray(integrality, dtype=bool)
        self.vmap = vmap
        self.fixed: dict = {}

    @property
    def n_rows(self) -> int:
        return self.lp.n_rows

    @property
    def n_cols(self) -> int:
        return self.lp.n_cols

    def relax(self) -> StandardFormLp:
        lp = self.lp
        return StandardFormLp(lp.matrix, lp.rhs.copy(), lp.cost.copy(), lp.lower.copy(),
                              lp.upper.copy(), lp.n_eq, lp.offset, list(lp.row_tags),
                              list(lp.col_tags))


_LAZY_CLASSES: dict = {}


def lazy_csc_matrix(cls, matrix):
    """An instance of ``cls`` -- the caller's ``SparseMatrix`` class, the
    reference's after ``install()`` -- holding the canonical CSR of `matrix`
    and building its CSC copy (and the CSR view of A^T) on first use.

    The reference's constructor converts to CSC eagerly
    (``lp_kernel.py:52-62``); the drop-in's model builder and presolve build
    large reduced models every fixing round, and the GPU engine only reads
    ``.csr`` (it transposes on the device), so the CSC conversion -- a few
    seconds at C4 -- is deferred until a CPU code path asks for it.  The
    object is an instance of ``cls`` and every attribute keeps its meaning;
    the CSC copy, when built, is the one ``cls`` would have built."""
    if cls is SparseMatrix:
        return SparseMatrix(matrix)
    sub = _LAZY_CLASSES.get(cls)
    if sub is None:
        def __init__(self, m, dtype=np.float64):
            import scipy.sparse as sp
            csr = sp.csr_matrix(m, dtype=dtype)
            csr.sum_duplicates()
            csr.eliminate_zeros()
            csr.sort_indices()
            self.csr = csr
            self.shape = csr.shape
            self.dtype = csr.dtype

        def _csc(self):
            c = self.__dict__.get("_lazy_csc")
            if c is None:
                c = self.csr.tocsc()
                c.sort_indices()
                self.__dict__["_lazy_csc"] = c
            return c

        sub = type(cls.__name__, (cls,), {
            "__init__": __init__,
            "csc": property(_csc),
            "_t": property(lambda self: _csc(self).T),
            # pickles (and copies through pickle) as the caller's own class
            "__reduce__": lambda self: (cls, (self.csr,)),
            "__module__": cls.__module__,
            "__doc__": cls.__doc__,
        })
        _LAZY_CLASSES[cls] = sub
    return sub(matrix)
