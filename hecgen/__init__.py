"""Seeded synthetic inputs shared by the oracle (``oracle/``) and the product
path (``paper_1606_00545_b200``).

This module holds none of the method's arithmetic: it builds canonical CSR
matrices (§2.1, the ``Ap``/``Aj``/``Ax`` arrays; int32 indices and
fp64 values, pinned by Table 2's Mb(CSR) column) and x vectors with
the shapes of the workloads in SURVEY.md §8(d).  Randomness is a counter-based
splitmix64 keyed by (seed, stream, index), implemented in ``hecgen.c``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hecgen.c")
_LIB = os.path.join(_HERE, "libhecgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile ``hecgen.c`` into ``libhecgen.so`` (gcc, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i32, i64, u64, dbl, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        lib.hecgen_ctr.restype = u64
        lib.hecgen_ctr.argtypes = [u64, u64, u64]
        lib.hecgen_u01.restype = dbl
        lib.hecgen_u01.argtypes = [u64, u64, u64]
        lib.hecgen_vector.restype = ctypes.c_int
        lib.hecgen_vector.argtypes = [i64, ctypes.c_int, u64, vp]
        lib.hecgen_poisson3d_nnz.restype = i64
        lib.hecgen_poisson3d_nnz.argtypes = [i32, i32, i32]
        lib.hecgen_poisson3d.restype = ctypes.c_int
        lib.hecgen_poisson3d.argtypes = [i32, i32, i32, vp, vp, vp]
        lib.hecgen_poisson2d_nnz.restype = i64
        lib.hecgen_poisson2d_nnz.argtypes = [i32, i32]
        lib.hecgen_poisson2d.restype = ctypes.c_int
        lib.hecgen_poisson2d.argtypes = [i32, i32, vp, vp, vp]
        lib.hecgen_powerlaw_rowptr.restype = i64
        lib.hecgen_powerlaw_rowptr.argtypes = [i32, i32, i32, dbl, u64, vp]
        lib.hecgen_powerlaw_fill.restype = ctypes.c_int
        lib.hecgen_powerlaw_fill.argtypes = [i32, i32, dbl, ctypes.c_int, u64, vp, vp, vp]
        lib.hecgen_degree_sort.restype = ctypes.c_int
        lib.hecgen_degree_sort.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp]
        lib.hecgen_spe10.restype = ctypes.c_int
        lib.hecgen_spe10.argtypes = [i32, i32, i32, u64, ctypes.POINTER(i32), ctypes.POINTER(i64),
                                     ctypes.POINTER(ctypes.POINTER(i32)), ctypes.POINTER(ctypes.POINTER(i32)),
                                     ctypes.POINTER(ctypes.POINTER(dbl))]
        lib.hecgen_random_rowptr.restype = i64
        lib.hecgen_random_rowptr.argtypes = [i32, i32, dbl, u64, vp]
        lib.hecgen_random_fill.restype = ctypes.c_int
        lib.hecgen_random_fill.argtypes = [i32, i32, dbl, ctypes.c_int, u64, vp, vp, vp]
        lib.hecgen_free.restype = None
        lib.hecgen_free.argtypes = [vp]
        lib.hecgen_fnv1a.restype = u64
        lib.hecgen_fnv1a.argtypes = [vp, i64, u64]
        _lib = lib
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


@dataclass
class Csr:
    """Canonical CSR container (no arithmetic). ``grid`` is (nx, ny, nz) for
    structured matrices (nz = 1 for 2D), else None."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # int32[n_rows+1]
    col: np.ndarray      # int32[nnz]
    val: np.ndarray      # float64[nnz]
    grid: tuple | None = None
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    def checksum(self) -> str:
        return fnv1a(self.row_ptr, self.col, self.val)


def fnv1a(*arrays) -> str:
    """FNV-1a over the raw bytes of the arrays, in order (run logs)."""
    lib = _load()
    h = 0
    for a in arrays:
        a = np.ascontiguousarray(a)
        h = lib.hecgen_fnv1a(_p(a), a.nbytes, h)
    return f"{h:016x}"


def checksum(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return f"{_load().hecgen_fnv1a(_p(a), a.nbytes, 0):016x}"


def ctr(seed: int, stream: int, index: int) -> int:
    return int(_load().hecgen_ctr(seed, stream, index))


def u01(seed: int, stream: int, index: int) -> float:
    return float(_load().hecgen_u01(seed, stream, index))


def vector(n: int, kind: str = "uniform", seed: int = 1606) -> np.ndarray:
    """x vectors: 'uniform' U[-1,1) (SURVEY §8(d) default), 'ones', 'int' in [-2^20, 2^20]."""
    kinds = {"uniform": 0, "ones": 1, "int": 2}
    x = np.empty(n, dtype=np.float64)
    if _load().hecgen_vector(n, kinds[kind], seed, _p(x)) != 0:
        raise ValueError("hecgen_vector failed")
    return x


def poisson3d(nx: int, ny: int, nz: int) -> Csr:
    """7-point Laplacian, diagonal 6, off-diagonals -1, Dirichlet truncation
    (PAPER §3.1 '3D_Poisson')."""
    lib = _load()
    nnz = lib.hecgen_poisson3d_nnz(nx, ny, nz)
    if nnz < 0:
        raise ValueError("bad grid")
    n = nx * ny * nz
    rp = np.empty(n + 1, np.int32)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    lib.hecgen_poisson3d(nx, ny, nz, _p(rp), _p(col), _p(val))
    return Csr(n, n, rp, col, val, grid=(nx, ny, nz), name=f"poisson3d_{nx}x{ny}x{nz}")


def poisson2d(nx: int, ny: int) -> Csr:
    """5-point Laplacian, diagonal 4, off-diagonals -1, Dirichlet truncation."""
    lib = _load()
    nnz = lib.hecgen_poisson2d_nnz(nx, ny)
    if nnz < 0:
        raise ValueError("bad grid")
    n = nx * ny
    rp = np.empty(n + 1, np.int32)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    lib.hecgen_poisson2d(nx, ny, _p(rp), _p(col), _p(val))
    return Csr(n, n, rp, col, val, grid=(nx, ny, 1), name=f"poisson2d_{nx}x{ny}")


POWERLAW_ALPHA = 2.171049  # gives mean row length 16.000 on [4, 2000]


def powerlaw(n: int, lmin: int = 4, lmax: int = 2000, alpha: float = POWERLAW_ALPHA,
             band: int = 4096, p_local: float = 0.9, integer_values: bool = False,
             seed: int = 545) -> Csr:
    """Power-law row-length matrix (SURVEY §8(d) 'Power-law recipe')."""
    lib = _load()
    rp = np.empty(n + 1, np.int32)
    nnz = lib.hecgen_powerlaw_rowptr(n, lmin, lmax, alpha, seed, _p(rp))
    if nnz < 0:
        raise ValueError("powerlaw: bad parameters or nnz overflow")
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    if lib.hecgen_powerlaw_fill(n, band, p_local, int(integer_values), seed, _p(rp), _p(col), _p(val)) != 0:
        raise ValueError("powerlaw fill failed")
    return Csr(n, n, rp, col, val, name=f"powerlaw_{n}{'_int' if integer_values else ''}")


def degree_sorted(A: Csr) -> Csr:
    """Degree-sorted stress variant (SURVEY §8(d) power-law recipe): the
    symmetric permutation P A P^T that puts rows in descending length order
    (stable), columns renamed with it and re-sorted.  Returns the matrix; its
    ``perm`` attribute holds perm[new] = old."""
    lib = _load()
    n = A.n_rows
    if A.n_cols != n:
        raise ValueError("degree_sorted: square matrices only")
    perm = np.empty(n, np.int32)
    rp = np.empty(n + 1, np.int32)
    col = np.empty(A.nnz, np.int32)
    val = np.empty(A.nnz, np.float64)
    if lib.hecgen_degree_sort(n, _p(A.row_ptr), _p(A.col), _p(A.val), _p(perm), _p(rp), _p(col), _p(val)) != 0:
        raise ValueError("degree_sorted failed")
    B = Csr(n, n, rp, col, val, name=f"{A.name}_dsorted")
    B.perm = perm
    return B


def spe10(nx: int = 60, ny: int = 220, nz: int = 85, seed: int = 10) -> Csr:
    """SPE10-shaped reservoir matrix (SURVEY §8(d) 'SPE10 recipe')."""
    lib = _load()
    n = ctypes.c_int32()
    nnz = ctypes.c_int64()
    rp = ctypes.POINTER(ctypes.c_int32)()
    col = ctypes.POINTER(ctypes.c_int32)()
    val = ctypes.POINTER(ctypes.c_double)()
    rc = lib.hecgen_spe10(nx, ny, nz, seed, ctypes.byref(n), ctypes.byref(nnz),
                          ctypes.byref(rp), ctypes.byref(col), ctypes.byref(val))
    if rc != 0:
        raise ValueError(f"spe10 failed ({rc})")
    try:
        a_rp = np.ctypeslib.as_array(rp, shape=(n.value + 1,)).copy()
        a_col = np.ctypeslib.as_array(col, shape=(max(nnz.value, 1),))[:nnz.value].copy()
        a_val = np.ctypeslib.as_array(val, shape=(max(nnz.value, 1),))[:nnz.value].copy()
    finally:
        for p in (rp, col, val):
            lib.hecgen_free(ctypes.cast(p, ctypes.c_void_p))
    return Csr(n.value, n.value, a_rp, a_col, a_val, name=f"spe10_{nx}x{ny}x{nz}")


def random_csr(n_rows: int, n_cols: int, density: float, integer_values: bool = False,
               seed: int = 7) -> Csr:
    """Small random sparse matrix (each entry present with probability density)."""
    lib = _load()
    rp = np.empty(n_rows + 1, np.int32)
    nnz = lib.hecgen_random_rowptr(n_rows, n_cols, density, seed, _p(rp))
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    lib.hecgen_random_fill(n_rows, n_cols, density, int(integer_values), seed, _p(rp), _p(col), _p(val))
    return Csr(n_rows, n_cols, rp, col, val, name=f"random_{n_rows}x{n_cols}")


def from_dense(a: np.ndarray) -> Csr:
    """Canonical CSR of a small dense array (stored entries = nonzeros)."""
    a = np.asarray(a, dtype=np.float64)
    rows, cols = np.nonzero(a)
    rp = np.zeros(a.shape[0] + 1, np.int32)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp).astype(np.int32)
    return Csr(a.shape[0], a.shape[1], rp, cols.astype(np.int32), a[rows, cols].copy())


def from_rows(n_cols: int, rows: list[list[tuple[int, float]]]) -> Csr:
    """CSR from explicit per-row (col, val) lists; kept as given (may be non-canonical)."""
    rp = [0]
    col, val = [], []
    for r in rows:
        for c, v in r:
            col.append(c)
            val.append(v)
        rp.append(len(col))
    return Csr(len(rows), n_cols, np.array(rp, np.int32), np.array(col, np.int32),
               np.array(val, np.float64))


# BASELINE.json configs.
CONFIGS = {
    "poisson2d_64": lambda: poisson2d(64, 64),
    "poisson3d_128": lambda: poisson3d(128, 128, 128),
    "poisson3d_256": lambda: poisson3d(256, 256, 256),
    "spe10": lambda: spe10(60, 220, 85),
    "powerlaw_8M": lambda: powerlaw(1 << 23),
    "poisson3d_150": lambda: poisson3d(150, 150, 150),  # the paper's own 3D_Poisson
    # SURVEY §8(d) secondary row: the power-law matrix with rows in descending length order
    "powerlaw_8M_dsorted": lambda: degree_sorted(powerlaw(1 << 23)),
}
