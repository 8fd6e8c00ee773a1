"""GPU parity of the SpMV consumers against the
oracle (oracle/krylov_ref.py): Eq. (2) fused epilogue, the vector operations of
Eqs. (3)-(6), BiCGSTAB (Alg. 4, M = I) and CG, on one GPU and through the
distributed entry points at P = 1."""
import numpy as np
import pytest

import hecgen
import oracle
from oracle import krylov_ref as K

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1606_00545_b200 as hec  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def dense(A):
    D = np.zeros((A.n_rows, A.n_cols))
    for i in range(A.n_rows):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            D[i, A.col[k]] = A.val[k]
    return D


@pytest.mark.parametrize("maker", [lambda: hecgen.random_csr(300, 300, 0.05, integer_values=True, seed=4),
                                   lambda: hecgen.powerlaw(5000, integer_values=True, seed=5)])
def test_spmv_axpby_integer_bitwise(maker):
    A = maker()
    x = hecgen.vector(A.n_cols, "int", seed=1)
    y0 = hecgen.vector(A.n_rows, "int", seed=2)
    M = hec.from_csr(A)
    for alpha, beta in [(1.0, 0.0), (2.0, -3.0), (-1.0, 1.0), (0.5, 0.25)]:
        yd = dev(y0)
        M.spmv_axpby(alpha, dev(x), beta, yd)
        torch.cuda.synchronize()
        ref = K.spmv_axpby(A, alpha, x, beta, y0)
        assert yd.cpu().numpy().tobytes() == ref.tobytes()


def test_spmv_axpby_beta_zero_ignores_y_and_float_tolerance():
    A = hecgen.spe10(20, 30, 10, seed=2)
    x = hecgen.vector(A.n_cols, "uniform", seed=3)
    y = torch.full((A.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    M = hec.from_csr(A)
    M.spmv_axpby(1.5, dev(x), 0.0, y)                 # beta = 0: y is not read
    ref = 1.5 * oracle.csr_spmv(A, x)
    got = y.cpu().numpy()
    assert np.all(np.abs(got - ref) <= 1.5 * oracle.tolerance(A, x))
    y0 = hecgen.vector(A.n_rows, "uniform", seed=4)
    yd = dev(y0)
    M.spmv_axpby(0.7, dev(x), -1.3, yd)
    ref = K.spmv_axpby(A, 0.7, x, -1.3, y0)
    tol = 0.7 * oracle.tolerance(A, x) + 1e-15 * (np.abs(ref) + 1.3 * np.abs(y0))
    assert np.all(np.abs(yd.cpu().numpy() - ref) <= tol)


def test_vector_ops():
    n = 100_003
    x = hecgen.vector(n, "uniform", seed=7)
    y = hecgen.vector(n, "uniform", seed=8)
    yd = dev(y)
    hec.axpby(2.5, dev(x), -0.5, yd)
    # the device contracts alpha x + beta y into one FMA: within 2u of the two-rounding oracle
    ref = K.axpby(2.5, x, -0.5, y)
    assert np.all(np.abs(yd.cpu().numpy() - ref) <= 2 * 2.0 ** -53 * (2.5 * np.abs(x) + 0.5 * np.abs(y)))
    zd = torch.empty(n, dtype=torch.float64, device="cuda")
    hec.axpbyz(1.0, dev(x), 0.0, dev(y), zd)
    assert zd.cpu().numpy().tobytes() == x.tobytes()
    assert hec.dot(dev(np.array([1.0, 2.0, 3.0])), dev(np.array([4.0, 5.0, 6.0]))) == 32.0
    d = hec.dot(dev(x), dev(y))
    bound = 2 * n * 2.0 ** -53 * float(np.sum(np.abs(x * y)))
    assert abs(d - K.dot(x, y)) <= bound
    xi = np.floor(hecgen.vector(n, "int", seed=9) / 1024.0)   # |xi| <= 2^10: every partial sum exact
    assert hec.dot(dev(xi), dev(xi)) == K.dot(xi, xi)
    assert abs(hec.norm2(dev(x)) - K.norm2(x)) <= 1e-14 * K.norm2(x)
    assert hec.dot(dev(x), dev(y)) == d                # deterministic: fixed order


def test_cg_poisson_matches_oracle():
    A = hecgen.poisson3d(20, 18, 16)
    b = hecgen.vector(A.n_rows, "uniform", seed=11)
    ref = K.cg(A, b, np.zeros(A.n_rows), 1e-10, 1000)
    M = hec.from_csr(A)
    xd = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
    info = M.cg(dev(b), xd, 1e-10, 1000)
    assert info.converged and ref.converged
    assert abs(info.iterations - ref.iterations) <= 1
    x = xd.cpu().numpy()
    assert np.linalg.norm(x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
    true_rel = np.linalg.norm(b - oracle.csr_spmv(A, x)) / np.linalg.norm(b)
    assert true_rel <= 2e-10 and abs(true_rel - info.rel_residual) <= 1e-11


def test_bicgstab_spe10_trajectory_matches_oracle():
    # Unpreconditioned BiCGSTAB does not converge on the SPE10-shaped matrix
    # (coefficients span ~1e-6..1e7; the paper pairs it with ILU, which is out of
    # scope): compare the first iterations' residual trajectory instead.
    A = hecgen.spe10(20, 30, 10, seed=2)
    b = hecgen.vector(A.n_rows, "uniform", seed=12)
    M = hec.from_csr(A)
    for it in (1, 3, 10):
        ref = K.bicgstab(A, b, np.zeros(A.n_rows), 1e-30, it)
        xd = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
        info = M.bicgstab(dev(b), xd, 1e-30, it)
        assert info.iterations == ref.iterations == it
        assert abs(info.rel_residual - ref.rel_residual) <= 1e-6 * ref.rel_residual


@pytest.mark.parametrize("maker,tol", [(lambda: hecgen.powerlaw(20000, seed=3), 1e-10),
                                       (lambda: hecgen.poisson2d(40, 30), 1e-10)])
def test_bicgstab_matches_oracle(maker, tol):
    A = maker()
    b = hecgen.vector(A.n_rows, "uniform", seed=12)
    ref = K.bicgstab(A, b, np.zeros(A.n_rows), tol, 2000)
    M = hec.from_csr(A)
    # (1) The residual trajectory follows the oracle's while the rounding
    # differences of the two summation orders (A5: any order is valid) are
    # still small.  On the power-law matrix they grow ~1e6x per 10 iterations
    # (measured: relative gap 1e-15 at k = 10, 7e-9 at k = 20, O(1) by k = 60,
    # scripts/bicg_traj.py), so only the first 20 iterations are compared.
    traj = K.bicgstab(A, b, np.zeros(A.n_rows), 1e-30, 20).history
    for k, rel in ((1, 1e-12), (5, 1e-12), (10, 1e-10), (20, 1e-5)):
        if k >= len(traj):
            break
        xd = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
        info = M.bicgstab(dev(b), xd, 1e-30, k)
        assert info.iterations == k
        assert abs(info.rel_residual - traj[k]) <= rel * traj[k], (k, info.rel_residual, traj[k])
    # (2) Converged solve: same outcome, a true residual within the tolerance
    # and the oracle's solution.  What A5 justifies stops at (1): past the
    # compared prefix BiCGSTAB's trajectory is rounding-chaotic (any valid
    # summation order is a different, equally correct run: 197 vs 170 on the
    # power-law matrix, 103 vs 101 on the 2D Poisson one), so the iteration
    # count is NOT pinned.  A stall fails `converged`; a premature stop fails
    # the true-residual bound.
    xd = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
    info = M.bicgstab(dev(b), xd, tol, 2000)
    assert info.converged == ref.converged and info.breakdown == ref.breakdown == 0
    x = xd.cpu().numpy()
    rel_true = np.linalg.norm(b - oracle.csr_spmv(A, x)) / np.linalg.norm(b)
    assert rel_true <= 5 * tol
    assert np.linalg.norm(x - ref.x) <= 1e3 * tol * np.linalg.norm(ref.x)


def test_bicgstab_identity_one_step_and_breakdown():
    I = hecgen.from_dense(np.eye(64))
    b = hecgen.vector(64, "uniform", seed=1)
    xd = torch.zeros(64, dtype=torch.float64, device="cuda")
    info = hec.from_csr(I).bicgstab(dev(b), xd, 1e-12, 10)
    assert info.converged and info.iterations == 1
    assert xd.cpu().numpy().tobytes() == b.tobytes()
    R = hecgen.from_dense(np.array([[0.0, 1.0], [-1.0, 0.0]]))
    xd = torch.zeros(2, dtype=torch.float64, device="cuda")
    info = hec.from_csr(R).bicgstab(dev(np.array([1.0, 0.0])), xd, 1e-14, 10)
    assert (info.breakdown, info.iterations, info.converged) == (3, 1, 0)


def test_breakdown_4_omega_and_cg_alpha_undefined():
    # the oracle's pinned examples (tests/test_oracle_krylov.py): (t, t) = 0 in
    # BiCGSTAB and (p, A p) = 0 in CG -> breakdown 4 at k = 1, x untouched
    A = hecgen.from_dense(np.array([[1.0, -1.0], [0.0, 0.0]]))
    xd = torch.zeros(2, dtype=torch.float64, device="cuda")
    info = hec.from_csr(A).bicgstab(dev(np.array([0.5, -0.5])), xd, 1e-14, 10)
    assert (info.breakdown, info.iterations, info.converged) == (4, 1, 0)
    assert xd.cpu().numpy().tolist() == [0.0, 0.0]
    B = hecgen.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]))
    xd = torch.zeros(2, dtype=torch.float64, device="cuda")
    info = hec.from_csr(B).cg(dev(np.array([1.0, 0.0])), xd, 1e-14, 10)
    assert (info.breakdown, info.iterations, info.converged) == (4, 1, 0)
    assert xd.cpu().numpy().tolist() == [0.0, 0.0]


def test_dist_solvers_single_rank_equal_single_gpu_bitwise():
    A = hecgen.poisson3d(16, 16, 12)
    b = hecgen.vector(A.n_rows, "uniform", seed=13)
    M = hec.from_csr(A)
    D = hec.Dist(A, hec.partition(A, 1), 0, None, 0)
    for method in ("cg", "bicgstab"):
        x1 = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
        x2 = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
        i1 = getattr(M, method)(dev(b), x1, 1e-9, 500)
        i2 = getattr(D, method)(dev(b), x2, 1e-9, 500)
        assert (i1.iterations, i1.converged) == (i2.iterations, i2.converged)
        assert x1.cpu().numpy().tobytes() == x2.cpu().numpy().tobytes()


def _group_solve(A, b, P, kind, method, tol, max_it, grid=None, p2p=False):
    plan = hec.partition(A, P, kind, grid)
    grp = hec.LocalDistGroup(A, plan, 0, None, p2p=p2p)
    pp = plan.part_ptr()
    bs = [dev(b[pp[p]:pp[p + 1]]) for p in range(P)]
    xs = [torch.zeros(int(pp[p + 1] - pp[p]), dtype=torch.float64, device="cuda") for p in range(P)]
    info = getattr(grp, method)(bs, xs, tol, max_it)
    x = np.concatenate([t.cpu().numpy() for t in xs])
    grp.free()
    return info, x


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("p2p", [False, True])
def test_cg_dist_p_ranks_emulated_matches_oracle(P, p2p):
    # hec_cg_dist's P > 1 logic (per-rank passes, the all-reduce of the dots,
    # identical scalar steps on every rank, hec_spmv_dist's exchange) on one
    # GPU: iteration count within +-1 of the oracle, its solution, a true
    # residual at the tolerance (SURVEY §8(f) NEXT-1 pins)
    A = hecgen.poisson3d(24, 20, 16)
    b = hecgen.vector(A.n_rows, "uniform", seed=21)
    ref = K.cg(A, b, np.zeros(A.n_rows), 1e-10, 1000)
    info, x = _group_solve(A, b, P, hec.PART_GRID, "cg", 1e-10, 1000, grid=(24, 20, 16), p2p=p2p)
    assert info.converged and ref.converged and info.breakdown == 0
    assert abs(info.iterations - ref.iterations) <= 1, (info.iterations, ref.iterations)
    assert np.linalg.norm(x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
    true_rel = np.linalg.norm(b - oracle.csr_spmv(A, x)) / np.linalg.norm(b)
    assert true_rel <= 2e-10 and abs(true_rel - info.rel_residual) <= 1e-11


@pytest.mark.parametrize("P", [4, 8])
def test_bicgstab_dist_p_ranks_emulated_matches_oracle(P):
    A = hecgen.powerlaw(20000, seed=3)
    b = hecgen.vector(A.n_rows, "uniform", seed=12)
    traj = K.bicgstab(A, b, np.zeros(A.n_rows), 1e-30, 10).history
    for k, rel in ((1, 1e-12), (5, 1e-12), (10, 1e-10)):
        info, _ = _group_solve(A, b, P, hec.PART_CONTIG_NNZ, "bicgstab", 1e-30, k)
        assert info.iterations == k
        assert abs(info.rel_residual - traj[k]) <= rel * traj[k], (k, info.rel_residual, traj[k])
    ref = K.bicgstab(A, b, np.zeros(A.n_rows), 1e-10, 2000)
    info, x = _group_solve(A, b, P, hec.PART_CONTIG_NNZ, "bicgstab", 1e-10, 2000, p2p=True)
    assert info.converged == ref.converged == 1 and info.breakdown == 0
    assert np.linalg.norm(b - oracle.csr_spmv(A, x)) / np.linalg.norm(b) <= 5e-10
    assert np.linalg.norm(x - ref.x) <= 1e-7 * np.linalg.norm(ref.x)


def test_dist_local_single_rank_equals_single_gpu_bitwise():
    A = hecgen.poisson3d(16, 16, 12)
    b = hecgen.vector(A.n_rows, "uniform", seed=13)
    M = hec.from_csr(A)
    for method in ("cg", "bicgstab"):
        x1 = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
        i1 = getattr(M, method)(dev(b), x1, 1e-9, 500)
        i2, x2 = _group_solve(A, b, 1, hec.PART_CONTIG_NNZ, method, 1e-9, 500)
        assert (i1.iterations, i1.converged) == (i2.iterations, i2.converged)
        assert x1.cpu().numpy().tobytes() == x2.tobytes()
