"""Conic program container shared by the oracle and the CUDA path.

Holds DATA ONLY (no arithmetic of the method).  The problem is PAPER.md:538-541
(§2, Eq. 1):

    min <c, x>  s.t.  G x - h in K_d^*,  l <= x_1 <= u,  x_2 in K_p

with x = (x_1 in R^{n1}, x_2 in R^{n2}).  Cone lists follow SPEC.md:22-32:
``pk/pdim`` are the primal blocks K_p over x[n1:n]; ``rk/rdim`` are the
constraint cones C_b (G x - h in C_b, i.e. the blocks of K_d^*), so the dual
y of block b lives in C_b^* (reading A1).
"""
from __future__ import annotations

import dataclasses

import numpy as np

# Cone kind codes (shared by include/pdcs.h, the oracle and the generators).
ZERO, NONNEG, SOC, RSOC, EXP, DUAL_EXP = 0, 1, 2, 3, 4, 5
KIND_NAMES = {ZERO: "zero", NONNEG: "nonneg", SOC: "soc", RSOC: "rsoc",
              EXP: "exp", DUAL_EXP: "dual_exp"}


@dataclasses.dataclass
class ConicProgram:
    m: int
    n: int
    n1: int
    row_ptr: np.ndarray   # int64 [m+1]
    col_idx: np.ndarray   # int32 [nnz], strictly increasing within a row
    vals: np.ndarray      # float64 [nnz]
    c: np.ndarray         # float64 [n]
    h: np.ndarray         # float64 [m]
    l: np.ndarray         # float64 [n1], -inf allowed
    u: np.ndarray         # float64 [n1], +inf allowed
    pk: np.ndarray        # int32 primal cone kinds over x[n1:]
    pdim: np.ndarray      # int64 primal cone dims
    rk: np.ndarray        # int32 row (constraint) cone kinds
    rdim: np.ndarray      # int64 row cone dims
    name: str = "program"
    # optional planted optimum (x*, y*, c^T x*) for generators that know it
    x_star: np.ndarray | None = None
    y_star: np.ndarray | None = None
    obj_star: float | None = None

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def n2(self) -> int:
        return self.n - self.n1

    def dense(self) -> np.ndarray:
        """Dense copy of G (small instances only)."""
        G = np.zeros((self.m, self.n))
        for i in range(self.m):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            G[i, self.col_idx[s:e]] = self.vals[s:e]
        return G

    def check(self) -> None:
        """Structural sanity (layout only; mirrors SPEC.md:41-49 checks)."""
        assert self.row_ptr.dtype == np.int64 and self.row_ptr.shape == (self.m + 1,)
        assert self.col_idx.dtype == np.int32 and self.vals.dtype == np.float64
        assert self.c.shape == (self.n,) and self.h.shape == (self.m,)
        assert self.l.shape == (self.n1,) and self.u.shape == (self.n1,)
        assert int(self.pdim.sum()) == self.n2, "primal cone dims must sum to n2"
        assert int(self.rdim.sum()) == self.m, "row cone dims must sum to m"


def csr_from_coo(m: int, n: int, rows: np.ndarray, cols: np.ndarray,
                 vals: np.ndarray):
    """Sort COO triplets into CSR (row-major, ascending column)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], np.asarray(vals, np.float64)[order]
    counts = np.bincount(rows, minlength=m)
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return row_ptr, cols.astype(np.int32), vals
