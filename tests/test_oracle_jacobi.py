"""Pins for the damped-Jacobi reference (oracle/jacobi_ref.py, A22).

Pinned against: the Laplacian eigenmode closed form (Jacobi on the 3D 7-point
operator scales the mode v_pqr by exactly 1 - omega*lambda/6), the fixed point
x* of A x* = b in exact integer arithmetic, exact rational brute force on tiny
matrices whose diagonal entries are powers of two, and convergence to
scipy's direct solve on a strictly diagonally dominant matrix."""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import hecgen
import oracle
from oracle import jacobi_ref as J


def dense(A):
    D = np.zeros((A.n_rows, A.n_cols))
    for i in range(A.n_rows):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col[k]] = A.val[k]
    return D


def test_diag_dense_and_missing_entries():
    A = hecgen.random_csr(40, 40, 0.15, seed=11)
    Dn = dense(A)
    d = J.diag(A)
    assert d.tolist() == np.diag(Dn).tolist()
    assert (d == 0).sum() > 5  # rows without a stored diagonal give +0.0
    with pytest.raises(ValueError):
        J.diag(hecgen.random_csr(4, 5, 0.5, seed=1))


@pytest.mark.parametrize("mode,omega", [((1, 1, 1), 2 / 3), ((2, 3, 1), 0.8), ((5, 7, 9), 1.0)])
def test_laplacian_eigenmode_contraction(mode, omega):
    # D = 6 I away from nothing (Dirichlet truncation keeps the diagonal 6), so
    # with b = 0 one sweep maps v to (I - omega/6 A) v = (1 - omega lambda / 6) v
    nx, ny, nz = 16, 12, 10
    p, q, r = mode
    A = hecgen.poisson3d(nx, ny, nz)
    I, Jg, K = np.meshgrid(np.arange(1, nx + 1), np.arange(1, ny + 1), np.arange(1, nz + 1), indexing="ij")
    v = (np.sin(p * math.pi * I / (nx + 1)) * np.sin(q * math.pi * Jg / (ny + 1))
         * np.sin(r * math.pi * K / (nz + 1))).transpose(2, 1, 0).reshape(-1)
    lam = 6 - 2 * math.cos(p * math.pi / (nx + 1)) - 2 * math.cos(q * math.pi / (ny + 1)) \
        - 2 * math.cos(r * math.pi / (nz + 1))
    d = J.diag(A)
    assert np.all(d == 6.0)
    b = np.zeros(A.n_rows)
    xn = J.jacobi(A, d, b, v, omega)
    assert np.all(np.abs(xn - (1 - omega * lam / 6) * v) <= 1e-13 * (np.abs(v) + 2 * oracle.csr_absmv(A, v)))
    assert np.all(np.abs(xn - (1 - omega * lam / 6) * v) <= J.tolerance(A, d, b, v, omega))


def test_fixed_point_integer_exact():
    # b = A x* computed exactly in integers: r = 0 exactly, so x* is returned bit for bit
    A = hecgen.spe10(12, 10, 5, seed=3)  # structure only (wells: long rows)
    rng = np.random.default_rng(4)
    vals = rng.integers(-8, 9, A.nnz).astype(np.float64)
    for i in range(A.n_rows):  # nonzero diagonal
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            if A.col[k] == i:
                vals[k] = 20.0
    A = hecgen.Csr(A.n_rows, A.n_cols, A.row_ptr, A.col, vals)
    xs = rng.integers(-1000, 1000, A.n_cols).astype(np.float64)
    b = (dense(A).astype(np.int64) @ xs.astype(np.int64)).astype(np.float64)
    for omega in (1.0, 2 / 3, 0.37):
        assert J.jacobi(A, J.diag(A), b, xs, omega).tobytes() == xs.tobytes()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_rational_bruteforce_power_of_two_diagonal(seed):
    # integer off-diagonals, diagonal in {+-2, +-4, +-8}, omega = 1/2: every step
    # (subtract, divide by a power of two, halve, add) is exact, so the sweep
    # must equal the rational-arithmetic result exactly
    rng = np.random.default_rng(seed)
    n = 25
    Dn = np.where(rng.random((n, n)) < 0.2, rng.integers(-8, 9, (n, n)), 0).astype(np.float64)
    np.fill_diagonal(Dn, rng.choice([-8, -4, -2, 2, 4, 8], n))
    A = hecgen.from_dense(Dn)
    x = rng.integers(-50, 50, n).astype(np.float64)
    b = rng.integers(-50, 50, n).astype(np.float64)
    got = J.jacobi(A, J.diag(A), b, x, 0.5)
    for i in range(n):
        ax = sum(Fraction(int(Dn[i, j])) * Fraction(int(x[j])) for j in range(n))
        want = Fraction(int(x[i])) + Fraction(1, 2) * (Fraction(int(b[i])) - ax) / Fraction(int(Dn[i, i]))
        assert Fraction(got[i]) == want


def test_converges_to_direct_solve():
    # strictly diagonally dominant (power-law generator: d_i = 1 + sum |off|):
    # Jacobi with omega = 1 converges to A^{-1} b
    A = hecgen.powerlaw(3000, lmin=3, lmax=40, band=64, seed=5)
    M = sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(A.n_rows, A.n_cols))
    b = hecgen.vector(A.n_rows, seed=6)
    xs = spla.spsolve(M.tocsc(), b)
    d = J.diag(A)
    x = np.zeros(A.n_rows)
    for _ in range(400):
        x = J.jacobi(A, d, b, x, 1.0)
    assert np.max(np.abs(x - xs)) <= 1e-9 * np.max(np.abs(xs))
