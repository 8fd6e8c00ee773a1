"""Pins for O1 / O1' / Eq. (1) (oracle/spmv_oracle.c, oracle/__init__.py).

Each test ties the oracle to something other than itself (SURVEY.md §8(c)
"What pins each part"): exact dense brute force, worked examples printed by
SPEC/the paper, Laplacian closed forms, and scipy as an independent library.
"""
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import hecgen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dense_exact(A, x):
    """Brute force with Python integers (exact) -- valid for integer data."""
    d = [[0] * A.n_cols for _ in range(A.n_rows)]
    for i in range(A.n_rows):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            d[i][int(A.col[k])] = int(A.val[k])
    return [sum(d[i][j] * int(x[j]) for j in range(A.n_cols)) for i in range(A.n_rows)]


@pytest.mark.parametrize("shape,density,seed", [((1, 1), 1.0, 1), ((7, 5), 0.5, 2), ((5, 9), 0.3, 3),
                                                ((33, 33), 0.2, 4), ((64, 64), 0.1, 5), ((64, 17), 0.9, 6)])
def test_o1_dense_bruteforce_integer_exact(shape, density, seed):
    # Integer entries in [-8,8], integer x in [-8,8]: every partial sum is an exact
    # integer < 2^53, so O1 must equal the dense product bit for bit.
    A = hecgen.random_csr(shape[0], shape[1], density, integer_values=True, seed=seed)
    x = np.array([(hecgen.ctr(seed, 99, j) % 17) - 8 for j in range(shape[1])], dtype=np.float64)
    y = oracle.csr_spmv(A, x)
    assert y.tolist() == [float(v) for v in dense_exact(A, x)]


def test_o1_nonsymmetric_catches_transpose():
    # A plausible bug (using A^T) must fail: non-symmetric 2x2 [[1,2],[3,4]] . [1,0] = [1,3].
    A = hecgen.from_dense([[1.0, 2.0], [3.0, 4.0]])
    assert oracle.csr_spmv(A, np.array([1.0, 0.0])).tolist() == [1.0, 3.0]


def test_o1_spec_hand_examples():
    # identity . x -> x ; [[1,2],[3,4]] . [1,1] -> [3,7]
    I = hecgen.from_dense(np.eye(4))
    x = np.array([0.5, -2.0, 3.25, 7.0])
    assert oracle.csr_spmv(I, x).tolist() == x.tolist()
    A = hecgen.from_dense([[1.0, 2.0], [3.0, 4.0]])
    assert oracle.csr_spmv(A, np.ones(2)).tolist() == [3.0, 7.0]
    # empty matrix (nnz = 0) -> zero vector
    E = hecgen.from_dense(np.zeros((3, 4)))
    assert E.nnz == 0
    assert oracle.csr_spmv(E, np.ones(4)).tolist() == [0.0, 0.0, 0.0]
    # 1x1x1 Poisson is [6]
    P1 = hecgen.poisson3d(1, 1, 1)
    assert oracle.csr_spmv(P1, np.ones(1)).tolist() == [6.0]


def test_o1_rectangular_and_row_range():
    A = hecgen.random_csr(5, 3, 0.7, integer_values=True, seed=11)
    x = np.array([1.0, -2.0, 3.0])
    full = oracle.csr_spmv(A, x)
    assert oracle.csr_spmv(A, x, 2, 5).tolist() == full[2:5].tolist()
    B = hecgen.random_csr(3, 5, 0.7, integer_values=True, seed=12)
    xb = np.arange(5, dtype=np.float64) - 2
    assert oracle.csr_spmv(B, xb).tolist() == [float(v) for v in dense_exact(B, xb)]


def test_eq1_column_view_equals_row_view():
    # PAPER Eq. (1): A x = sum_k x_k A[:,k]; exact on integer data,
    # within tau on random data.
    A = hecgen.random_csr(40, 40, 0.2, integer_values=True, seed=21)
    x = np.array([(j % 9) - 4 for j in range(40)], dtype=np.float64)
    assert oracle.column_spmv(A, x).tolist() == oracle.csr_spmv(A, x).tolist()
    B = hecgen.random_csr(50, 50, 0.3, seed=22)
    xb = hecgen.vector(50, "uniform", seed=3)
    d = np.abs(oracle.column_spmv(B, xb) - oracle.csr_spmv(B, xb))
    assert np.all(d <= oracle.tolerance(B, xb))


def test_o1_scipy_crosscheck():
    # Reduces to a library routine: scipy.sparse CSR matvec, within tau.
    for A in (hecgen.random_csr(100, 100, 0.05, seed=31), hecgen.spe10(12, 20, 9, seed=4),
              hecgen.powerlaw(3000, seed=5)):
        x = hecgen.vector(A.n_cols, "uniform", seed=7)
        S = sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(A.n_rows, A.n_cols))
        d = np.abs(S @ x - oracle.csr_spmv(A, x))
        assert np.all(d <= oracle.tolerance(A, x) + 0.0)


def test_o1_parallel_is_bit_identical():
    # O1p (OpenMP rows, timing only) must be O1 bit for bit: one thread per row, same order
    for A in (hecgen.powerlaw(50000, seed=2), hecgen.spe10(20, 30, 10, seed=1), hecgen.poisson3d(30, 20, 10)):
        x = hecgen.vector(A.n_cols, "uniform", seed=3)
        y, threads = oracle.csr_spmv_parallel(A, x)
        assert threads >= 1
        assert y.tobytes() == oracle.csr_spmv(A, x).tobytes()


def test_o1_dense_random_1e13():
    # random 100x100 at 5% vs dense matvec to 1e-13 relative.
    A = hecgen.random_csr(100, 100, 0.05, seed=41)
    D = np.zeros((100, 100))
    for i in range(100):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col[k]] = A.val[k]
    x = hecgen.vector(100, "uniform", seed=42)
    y = oracle.csr_spmv(A, x)
    assert np.all(np.abs(y - D @ x) <= 1e-13 * (np.abs(D) @ np.abs(x)))


def _degree_3d(nx, ny, nz):
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    deg = (i > 0).astype(int) + (i < nx - 1) + (j > 0) + (j < ny - 1) + (k > 0) + (k < nz - 1)
    return deg.transpose(2, 1, 0).reshape(-1)     # natural order i + nx*(j + ny*k)


@pytest.mark.parametrize("dims", [(16, 12, 10), (3, 3, 3), (1, 5, 2), (7, 1, 1)])
def test_p1_laplacian_constant_vector_3d(dims):
    # P1: (A 1)_i = 6 - deg(i) exactly (0 on interior rows); (|A||1|)_i = 6 + deg(i).
    A = hecgen.poisson3d(*dims)
    deg = _degree_3d(*dims)
    y = oracle.csr_spmv(A, np.ones(A.n_cols))
    assert y.tolist() == (6 - deg).astype(float).tolist()
    r = oracle.csr_absmv(A, np.ones(A.n_cols))
    assert r.tolist() == (6 + deg).astype(float).tolist()


def test_p1_laplacian_constant_vector_2d():
    nx, ny = 64, 64
    A = hecgen.poisson2d(nx, ny)
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    deg = ((i > 0).astype(int) + (i < nx - 1) + (j > 0) + (j < ny - 1)).reshape(-1)
    assert oracle.csr_spmv(A, np.ones(A.n_cols)).tolist() == (4 - deg).astype(float).tolist()


@pytest.mark.parametrize("mode", [(1, 1, 1), (2, 3, 1), (5, 7, 9), (16, 12, 10)])
def test_p2_laplacian_sine_eigenmodes(mode):
    # P2: v_pqr = sin(p pi i/(nx+1)) sin(q pi j/(ny+1)) sin(r pi k/(nz+1)) (1-based),
    # lambda = 6 - 2cos(p pi/(nx+1)) - 2cos(q pi/(ny+1)) - 2cos(r pi/(nz+1)).
    nx, ny, nz = 16, 12, 10
    p, q, r = mode
    A = hecgen.poisson3d(nx, ny, nz)
    I, J, K = np.meshgrid(np.arange(1, nx + 1), np.arange(1, ny + 1), np.arange(1, nz + 1), indexing="ij")
    v = (np.sin(p * math.pi * I / (nx + 1)) * np.sin(q * math.pi * J / (ny + 1))
         * np.sin(r * math.pi * K / (nz + 1))).transpose(2, 1, 0).reshape(-1)
    lam = 6 - 2 * math.cos(p * math.pi / (nx + 1)) - 2 * math.cos(q * math.pi / (ny + 1)) \
        - 2 * math.cos(r * math.pi / (nz + 1))
    y = oracle.csr_spmv(A, v)
    assert np.all(np.abs(y - lam * v) <= 1e-13 * oracle.csr_absmv(A, v))


def test_p4_poisson_sizes_printed_in_paper():
    for line in open(os.path.join(GOLD, "poisson_sizes.txt")):
        if line.startswith("#") or not line.strip():
            continue
        nx, ny, nz, rows, nnz = (int(t) for t in line.split()[:5])
        if nx * ny * nz <= 200000:
            A = hecgen.poisson3d(nx, ny, nz)
            assert (A.n_rows, A.nnz) == (rows, nnz)
        else:
            assert nx * ny * nz == rows
            assert hecgen._load().hecgen_poisson3d_nnz(nx, ny, nz) == nnz


def test_p4_nnz_closed_form_random_shapes():
    # nnz = 7n - 2(ny nz + nx nz + nx ny), 10 shapes.
    for s in range(10):
        nx, ny, nz = (1 + hecgen.ctr(s, 50, t) % 20 for t in range(3))
        n = nx * ny * nz
        assert hecgen._load().hecgen_poisson3d_nnz(nx, ny, nz) == 7 * n - 2 * (ny * nz + nx * nz + nx * ny)
    # BASELINE configs: 64^2 -> 4096/20224; 128^3 -> 2097152/14581760; 256^3 -> 16777216/117047296
    assert hecgen._load().hecgen_poisson2d_nnz(64, 64) == 20224
    assert hecgen._load().hecgen_poisson3d_nnz(128, 128, 128) == 14581760
    assert hecgen._load().hecgen_poisson3d_nnz(256, 256, 256) == 117047296


def test_a8_table2_byte_model():
    # Reading A8: the paper's CSR is fp64 + int32 + int32 row pointers, since
    # Mb(CSR) = round((12 nnz + 4 (n+1)) / 2^20) for all 12 matrices of Table 2.
    rows = [l.split() for l in open(os.path.join(GOLD, "paper_table2.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 12
    for name, n, nnz, per, mb in rows:
        n, nnz, per, mb = int(n), int(nnz), int(per), int(mb)
        assert round((12 * nnz + 4 * (n + 1)) / 2 ** 20) == mb, name
        assert round(nnz / n) == per, name


def test_tolerance_bound_is_order_independent():
    # two summation orders of a length-m dot product differ by at
    # most 2 gamma_m (|A||x|)_i; 2 m u <= 1e-12 for m <= 4503 (powerlaw max 2000).
    u = 2.0 ** -53
    assert 2 * 4503 * u <= 1e-12
    assert 2 * 4504 * u > 1e-12 * 0.99


def test_is_canonical_rejects_bad_inputs():
    good = hecgen.from_dense([[1.0, 0, 2.0], [0, 3.0, 0]])
    assert oracle.is_canonical(good)
    assert not oracle.is_canonical(hecgen.from_rows(3, [[(2, 1.0), (0, 1.0)]]))   # unsorted
    assert not oracle.is_canonical(hecgen.from_rows(3, [[(1, 1.0), (1, 1.0)]]))   # duplicate
    assert not oracle.is_canonical(hecgen.from_rows(3, [[(3, 1.0)]]))             # out of range
