"""Damped-Jacobi sweep -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY.md §8(f) NEXT-3, second epilogue: the smoother the paper's AMG uses
("The smoothers include damped Jacobi and weighted Jacobi"; "The
dJacobi, wJacobi and Chev are all developed based on the SpMV and vector
operations").  The paper prints no formula; reading A22 takes
the textbook damped-Jacobi step

    x_new = x + omega * D^{-1} (b - A x),     D = diag(A)

evaluated in this order: r = b - A x (A x is O1), then q_i = r_i / d_i, then
x_new_i = x_i + omega * q_i, every operation rounded on its own (no FMA).

  diag(A)     d_i = the stored entry A_ii, +0.0 when row i stores none
  jacobi      one sweep
  tolerance   |x_gpu - x_ref|_i <= 1e-12 (|x_i| + |omega/d_i| (|b_i| + (|A||x|)_i))
              (A22: the 1e-12 (|A||x|)_i bound of the SpMV carried
              through the subtraction, division, scaling and addition)

Pins: tests/test_oracle_jacobi.py (Laplacian eigenmode contraction factor,
fixed point in the integer regime, convergence to scipy's direct solve,
dense brute force on tiny integer matrices).
"""
from __future__ import annotations

import numpy as np

from . import csr_absmv, csr_spmv


def diag(A, r0: int = 0, r1: int | None = None) -> np.ndarray:
    """d_i = A_ii if row i stores column i, else +0.0 (square A); rows [r0, r1)."""
    if A.n_rows != A.n_cols:
        raise ValueError("diag needs a square matrix")
    r1 = A.n_rows if r1 is None else r1
    d = np.zeros(r1 - r0, dtype=np.float64)
    for i in range(r0, r1):
        for k in range(int(A.row_ptr[i]), int(A.row_ptr[i + 1])):
            if int(A.col[k]) == i:
                d[i - r0] = A.val[k]
    return d


def jacobi(A, d: np.ndarray, b: np.ndarray, x: np.ndarray, omega: float,
           r0: int = 0, r1: int | None = None) -> np.ndarray:
    """One damped-Jacobi sweep x + omega D^{-1} (b - A x), rows [r0, r1).
    d and b hold rows [r0, r1); x is the whole vector."""
    r1 = A.n_rows if r1 is None else r1
    r = b - csr_spmv(A, x, r0, r1)   # numpy elementwise: one rounding each
    q = r / d
    return x[r0:r1] + omega * q


def tolerance(A, d: np.ndarray, b: np.ndarray, x: np.ndarray, omega: float,
              r0: int = 0, r1: int | None = None) -> np.ndarray:
    r1 = A.n_rows if r1 is None else r1
    with np.errstate(divide="ignore", invalid="ignore"):
        g = np.abs(omega / d)
    return 1e-12 * (np.abs(x[r0:r1]) + g * (np.abs(b) + csr_absmv(A, x, r0, r1)))
