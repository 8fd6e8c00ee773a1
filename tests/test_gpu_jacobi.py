"""GPU parity of hec_diag / hec_jacobi (the damped-Jacobi
epilogue, A22) against oracle/jacobi_ref.py, through the C ABI.

Bar: hec_diag bit-exact; the sweep within 1e-12 (|x_i| + |omega/d_i| (|b_i| +
(|A||x|)_i)); bitwise where every operation is exact (integer data, power-of-two
diagonal, omega = 1/2) and, for rows without a tail, wherever the oracle's four
roundings are the kernel's (integer data, any d, any omega)."""
import numpy as np
import pytest
import hecgen
import oracle
from oracle import jacobi_ref as J

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1606_00545_b200 as hec  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def nan_vec(n):
    return torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")


def gpu_diag(M, n):
    d = nan_vec(n)
    M.diag(d)
    torch.cuda.synchronize()
    return d


MAKERS = [
    ("poisson2d_64", lambda: hecgen.poisson2d(64, 64), None),
    ("poisson3d_32", lambda: hecgen.poisson3d(32, 32, 32), None),
    ("spe10", lambda: hecgen.spe10(60, 220, 85), None),             # wells: diagonal in the tail
    ("powerlaw_64k", lambda: hecgen.powerlaw(1 << 16), None),
    ("random_missing_diag", lambda: hecgen.random_csr(700, 700, 0.01, seed=5), None),
    ("all_tail", lambda: hecgen.powerlaw(5000, seed=3), (hec.WIDTH_CAP, 0)),
    ("spe10_hyb", lambda: hecgen.spe10(20, 30, 10, seed=2), "hyb"),
]


def build(A, how):
    if how == "hyb":
        return hec.from_csr_hyb(A)
    return hec.from_csr(A, hec.opts(*how) if how else None)


@pytest.mark.parametrize("name,maker,how", MAKERS)
def test_diag_bitexact(name, maker, how):
    A = maker()
    M = build(A, how)
    d = gpu_diag(M, A.n_rows).cpu().numpy()
    assert d.tobytes() == J.diag(A).tobytes()
    if name == "spe10":
        assert M.info.tail_rows > 0


@pytest.mark.parametrize("name,maker,how", [m for m in MAKERS if m[0] != "random_missing_diag"])
@pytest.mark.parametrize("omega", [1.0, 2 / 3])
def test_sweep_within_tolerance(name, maker, how, omega):
    A = maker()
    M = build(A, how)
    x = hecgen.vector(A.n_rows, "uniform", seed=21)
    b = hecgen.vector(A.n_rows, "uniform", seed=22)
    d = J.diag(A)
    out = nan_vec(A.n_rows)
    M.jacobi(gpu_diag(M, A.n_rows), dev(b), dev(x), out, omega)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    ref = J.jacobi(A, d, b, x, omega)
    tol = J.tolerance(A, d, b, x, omega)
    bad = np.nonzero(~(np.abs(got - ref) <= tol))[0]
    assert bad.size == 0, f"{bad.size} rows out of tolerance, first {bad[:5]}: {got[bad[:5]]} vs {ref[bad[:5]]}"


@pytest.mark.parametrize("maker", [lambda: hecgen.poisson2d(64, 64), lambda: hecgen.poisson3d(40, 33, 17)])
def test_integer_data_no_tail_bitwise(maker):
    # no tail: the kernel's r = b - s, q = r / d, x + omega q are the oracle's roundings
    A = maker()
    M = hec.from_csr(A)
    assert M.info.tail_rows == 0
    x = hecgen.vector(A.n_rows, "int", seed=3)
    b = hecgen.vector(A.n_rows, "int", seed=4)
    d = J.diag(A)
    for omega in (1.0, 2 / 3, 0.8):
        out = nan_vec(A.n_rows)
        M.jacobi(dev(d), dev(b), dev(x), out, omega)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == J.jacobi(A, d, b, x, omega).tobytes()


def test_exact_regime_with_tail_bitwise():
    # SPE10 structure (well rows spill into the tail), integer off-diagonals,
    # diagonal 16, omega = 1/2, small integer x, b: every operation on both
    # sides is exact, so the split ELL/tail update must match bit for bit
    A = hecgen.spe10(30, 40, 12, seed=4)
    rng = np.random.default_rng(8)
    vals = rng.integers(-8, 9, A.nnz).astype(np.float64)
    for i in range(A.n_rows):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            if A.col[k] == i:
                vals[k] = 16.0
    A = hecgen.Csr(A.n_rows, A.n_cols, A.row_ptr, A.col, vals)
    M = hec.from_csr(A)
    assert M.info.tail_rows > 0
    x = rng.integers(-64, 64, A.n_rows).astype(np.float64)
    b = rng.integers(-64, 64, A.n_rows).astype(np.float64)
    d = J.diag(A)
    out = nan_vec(A.n_rows)
    M.jacobi(gpu_diag(M, A.n_rows), dev(b), dev(x), out, 0.5)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == J.jacobi(A, d, b, x, 0.5).tobytes()


def test_sweeps_converge():
    # the smoother as a solver: strictly diagonally dominant power-law matrix
    # (d_i = 1 + sum |off|) with long rows in the tail; 400 ping-pong sweeps
    # drive the residual b - A x (oracle O1) to rounding level
    A = hecgen.powerlaw(1 << 15, lmin=3, lmax=40, band=64, seed=9)
    M = hec.from_csr(A)
    assert M.info.tail_rows > 0
    b = hecgen.vector(A.n_rows, "uniform", seed=10)
    d = gpu_diag(M, A.n_rows)
    bd = dev(b)
    u, v = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda"), nan_vec(A.n_rows)
    for _ in range(400):
        M.jacobi(d, bd, u, v, 1.0)
        u, v = v, u
    torch.cuda.synchronize()
    x = u.cpu().numpy()
    assert np.max(np.abs(b - oracle.csr_spmv(A, x))) <= 1e-10 * np.max(np.abs(b))


def test_errors():
    R = hec.from_csr(hecgen.random_csr(30, 20, 0.2, seed=1))
    v = nan_vec(30)
    with pytest.raises(hec.HecError) as e:
        R.diag(v)
    assert e.value.status == 3
    A = hecgen.poisson2d(8, 8)
    M = hec.from_csr(A)
    x = dev(np.ones(64))
    with pytest.raises(hec.HecError) as e:
        M.jacobi(x, x, x, x, 1.0)  # x_out overlaps x
    assert e.value.status == 1
