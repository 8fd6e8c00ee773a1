"""oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct CPU statement of what the HEC SpMV hot path
computes, written from PAPER.md (arXiv 1606.00545) and the readings in
SURVEY.md §8(c) / DESIGN.md.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import it.
The product package ``paper_1606_00545_b200`` never imports, links or executes
anything under ``oracle/`` and shares no code with it; the only common module
is ``hecgen`` (seeded input generators, no method arithmetic).

Contents (SURVEY.md §8(c) names):
  O1  csr_spmv      serial CSR y = A x, column order, no FMA   (spmv_oracle.c)
  O1p csr_spmv_parallel  the same rows over OpenMP threads (bit-identical; timing only)
  O1' csr_absmv     (|A||x|)_i, the tolerance scale           (spmv_oracle.c)
  Eq1 column_spmv   y = sum_k x_k A[:,k]  (Eq. (1))  (numpy, column order)
  O2  hec_ref       HEC reference builder                     (hec_ref.py)
  O3  plan_ref      partition + halo plan reference           (plan_ref.py)
  O4  dist_ref      distributed result + simulated exchange   (plan_ref.py)

Pins (tests/test_oracle_*.py) tie each function to something other than
itself: dense brute force in the integer-exact regime, the paper's printed
Poisson sizes, Laplacian closed forms, SPEC worked examples, scipy.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spmv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

TOL_REL = 1e-12  # |y_gpu - y_ref|_i <= 1e-12 (|A||x|)_i  (BASELINE.json north_star)


def build(force: bool = False) -> str:
    """Compile the C oracle: -O2 -ffp-contract=off -fno-fast-math (no FMA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i32, vp = ctypes.c_int32, ctypes.c_void_p
        for f in (lib.oracle_csr_spmv, lib.oracle_csr_absmv):
            f.restype = None
            f.argtypes = [i32, i32, vp, vp, vp, vp, vp]
        lib.oracle_csr_spmv_omp.restype = ctypes.c_int
        lib.oracle_csr_spmv_omp.argtypes = [i32, i32, vp, vp, vp, vp, vp]
        _lib = lib
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def _arrays(A):
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int32)
    col = np.ascontiguousarray(A.col, dtype=np.int32)
    val = np.ascontiguousarray(A.val, dtype=np.float64)
    return rp, col, val


def csr_spmv(A, x: np.ndarray, r0: int = 0, r1: int | None = None) -> np.ndarray:
    """O1: y_i = sum_k val[k] * x[col[k]] in column order, products rounded
    then added (Eq. (1); Alg. 1).  Rows [r0, r1)."""
    r1 = A.n_rows if r1 is None else r1
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.shape[0] == A.n_cols
    rp, col, val = _arrays(A)
    y = np.empty(r1 - r0, dtype=np.float64)
    _load().oracle_csr_spmv(r0, r1, _p(rp), _p(col), _p(val), _p(x), _p(y))
    return y


def csr_spmv_parallel(A, x: np.ndarray) -> tuple[np.ndarray, int]:
    """O1 with its rows split over host threads (OpenMP):
    bit-identical to csr_spmv, for timing a parallel CPU baseline.  Returns
    (y, threads used)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.shape[0] == A.n_cols
    rp, col, val = _arrays(A)
    y = np.empty(A.n_rows, dtype=np.float64)
    t = _load().oracle_csr_spmv_omp(0, A.n_rows, _p(rp), _p(col), _p(val), _p(x), _p(y))
    return y, int(t)


def csr_absmv(A, x: np.ndarray, r0: int = 0, r1: int | None = None) -> np.ndarray:
    """O1': r_i = sum_k |val[k]| |x[col[k]]| -- the scale of the tolerance."""
    r1 = A.n_rows if r1 is None else r1
    x = np.ascontiguousarray(x, dtype=np.float64)
    rp, col, val = _arrays(A)
    r = np.empty(r1 - r0, dtype=np.float64)
    _load().oracle_csr_absmv(r0, r1, _p(rp), _p(col), _p(val), _p(x), _p(r))
    return r


def column_spmv(A, x: np.ndarray) -> np.ndarray:
    """Eq. (1): A x = x_1 A[:,1] + x_2 A[:,2] + ... ,
    accumulated column by column (a different summation order from O1)."""
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
    order = np.lexsort((rows, A.col))          # entries grouped by column
    y = np.zeros(A.n_rows, dtype=np.float64)
    for k in order:                             # plain loop: small inputs only
        y[rows[k]] = y[rows[k]] + A.val[k] * x[A.col[k]]
    return y


def tolerance(A, x: np.ndarray, r0: int = 0, r1: int | None = None) -> np.ndarray:
    """tau_i = 1e-12 (|A||x|)_i (BASELINE.json north_star)."""
    return TOL_REL * csr_absmv(A, x, r0, r1)


def is_canonical(A) -> bool:
    """SPEC S:31-35 / SURVEY §8(c) A7: row_ptr[0]=0, non-decreasing,
    row_ptr[n]=nnz, strictly increasing columns per row, 0 <= col < n_cols."""
    rp = np.asarray(A.row_ptr, dtype=np.int64)
    if rp.shape[0] != A.n_rows + 1 or rp[0] != 0 or rp[-1] != len(A.col):
        return False
    if np.any(np.diff(rp) < 0):
        return False
    for i in range(A.n_rows):
        c = np.asarray(A.col[rp[i]:rp[i + 1]], dtype=np.int64)
        if c.size and (c.min() < 0 or c.max() >= A.n_cols or np.any(np.diff(c) <= 0)):
            return False
    return True


from . import hec_ref, plan_ref, krylov_ref, reorder_ref, jacobi_ref  # noqa: E402,F401
