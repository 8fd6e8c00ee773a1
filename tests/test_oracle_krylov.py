"""Pins for the vector-operation and Krylov references (oracle/krylov_ref.py).

Pinned against: SPEC's worked examples, closed forms, exact integer
arithmetic, the finite-termination property of CG in exact arithmetic (at most
#distinct-eigenvalues iterations), and a library solve (numpy.linalg.solve)."""
import math

import numpy as np
import pytest

import hecgen
import oracle
from oracle import krylov_ref as K


def test_vector_ops_spec_examples():
    # axpbyz(1, x, 0, y) -> x ; dot([1,2,3],[4,5,6]) -> 32
    x = np.array([1.0, 2.0, 3.0])
    y = np.array([4.0, 5.0, 6.0])
    assert K.axpbyz(1.0, x, 0.0, y).tolist() == x.tolist()
    assert K.dot(x, y) == 32.0
    assert K.norm2(np.array([3.0, 4.0])) == 5.0
    assert K.axpby(2.0, x, -1.0, y).tolist() == [-2.0, -1.0, 0.0]


def test_spmv_axpby_integer_exact():
    A = hecgen.random_csr(30, 30, 0.2, integer_values=True, seed=3)
    x = np.arange(30, dtype=np.float64) - 15
    y = (np.arange(30, dtype=np.float64) % 7) - 3
    D = np.zeros((30, 30))
    for i in range(30):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col[k]] = A.val[k]
    assert K.spmv_axpby(A, 3.0, x, -2.0, y).tolist() == (3.0 * (D @ x) - 2.0 * y).tolist()


def test_cg_finite_termination_diagonal():
    # SPD diagonal matrix with 4 distinct eigenvalues: CG terminates in <= 4 steps.
    d = np.array([1.0, 2.0, 3.0, 4.0] * 10)
    A = hecgen.from_dense(np.diag(d))
    b = np.ones(40)
    res = K.cg(A, b, np.zeros(40), 1e-12, 100)
    assert res.converged and res.iterations <= 4
    assert np.allclose(res.x, b / d, rtol=1e-12)


def test_cg_matches_library_solve_on_poisson():
    A = hecgen.poisson3d(6, 5, 4)
    b = hecgen.vector(A.n_rows, "uniform", seed=2)
    res = K.cg(A, b, np.zeros(A.n_rows), 1e-12, 500)
    D = np.zeros((A.n_rows, A.n_rows))
    for i in range(A.n_rows):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col[k]] = A.val[k]
    xs = np.linalg.solve(D, b)
    assert res.converged
    assert np.linalg.norm(res.x - xs) <= 1e-9 * np.linalg.norm(xs)
    # the recurrence residual tracks the true residual
    true_rel = np.linalg.norm(b - D @ res.x) / np.linalg.norm(b)
    assert true_rel <= 1e-11 and abs(true_rel - res.rel_residual) <= 1e-11


def test_bicgstab_identity_and_exact_guess():
    I = hecgen.from_dense(np.eye(5))
    b = np.array([1.0, -2.0, 3.0, 0.5, 4.0])
    res = K.bicgstab(I, b, np.zeros(5), 1e-12, 10)
    assert res.converged and res.iterations == 1 and res.x.tolist() == b.tolist()   # s = 0 after one step
    res = K.bicgstab(I, b, b.copy(), 1e-12, 10)                                      # r0 = 0
    assert res.converged and res.iterations == 0


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_bicgstab_nonsymmetric_matches_library_solve(seed):
    # diagonally dominant nonsymmetric matrix (the power-law recipe's values)
    A = hecgen.powerlaw(300, seed=seed)
    b = hecgen.vector(300, "uniform", seed=seed)
    res = K.bicgstab(A, b, np.zeros(300), 1e-12, 300)
    D = np.zeros((300, 300))
    for i in range(300):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col[k]] = A.val[k]
    xs = np.linalg.solve(D, b)
    assert res.converged and res.breakdown == 0
    assert np.linalg.norm(res.x - xs) <= 1e-10 * np.linalg.norm(xs)
    assert np.linalg.norm(b - D @ res.x) <= 1e-11 * np.linalg.norm(b)


def test_bicgstab_on_spd_poisson_agrees_with_cg_solution():
    A = hecgen.poisson2d(12, 9)
    b = hecgen.vector(A.n_rows, "uniform", seed=5)
    r1 = K.bicgstab(A, b, np.zeros(A.n_rows), 1e-12, 500)
    r2 = K.cg(A, b, np.zeros(A.n_rows), 1e-12, 500)
    assert r1.converged and r2.converged
    assert np.linalg.norm(r1.x - r2.x) <= 1e-9 * np.linalg.norm(r2.x)


def test_bicgstab_breakdown_pivot():
    # A = [[0,1],[-1,0]] (rotation), b = e1: v = A r0 = -e2 is orthogonal to
    # r0 = e1, so alpha = rho / (r0, v) is undefined -> breakdown 3 at k = 1.
    A = hecgen.from_dense(np.array([[0.0, 1.0], [-1.0, 0.0]]))
    res = K.bicgstab(A, np.array([1.0, 0.0]), np.zeros(2), 1e-14, 10)
    assert (res.breakdown, res.iterations, res.converged) == (3, 1, False)


def test_bicgstab_breakdown_omega_undefined():
    # A = [[1, -1], [0, 0]]: u = e1 is an eigenvector (lambda 1), w = (1, 1) spans
    # the null space.  With r0 = u + c w, alpha_1 = (r,r)/(r,Ar) = 1/lambda exactly
    # when w.(w + u) = 0, i.e. c = -1/2, and then t = A s = A r - alpha A^2 r = 0
    # with s = (-1/2, -1/2) != 0: (t, t) = 0, omega_1 undefined -> breakdown 4
    # (reading A20).  Every value is a dyadic rational: exact in fp64.
    A = hecgen.from_dense(np.array([[1.0, -1.0], [0.0, 0.0]]))
    res = K.bicgstab(A, np.array([0.5, -0.5]), np.zeros(2), 1e-14, 10)
    assert (res.breakdown, res.iterations, res.converged) == (4, 1, False)
    assert res.x.tolist() == [0.0, 0.0]                  # no update with an undefined omega


def test_cg_breakdown_indefinite():
    # A = [[0, 1], [1, 0]] (symmetric, indefinite), b = e1: p = r = e1, A p = e2,
    # (p, A p) = 0 -> alpha undefined -> breakdown 4 at k = 1.
    A = hecgen.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]))
    res = K.cg(A, np.array([1.0, 0.0]), np.zeros(2), 1e-14, 10)
    assert (res.breakdown, res.iterations, res.converged) == (4, 1, False)
    assert res.x.tolist() == [0.0, 0.0]
