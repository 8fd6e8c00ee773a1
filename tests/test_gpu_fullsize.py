"""Full-size GPU parity, EVERY row against the serial C oracle O1,
at BASELINE.json's sizes and in the launch configuration bench.py times.

- configs[2] poisson3d_256 (16.8 M rows): hec_spmv with uniform x (tolerance),
  ones (closed form A 1 = 6 - deg, bitwise) and integer x (bitwise); the
  8-slab partition of the scaling run through both emulated transports
  (device copies and the peer-memory push kernel).
- configs[4] powerlaw_8M (8.4 M rows, 2.6 M tail rows, 79 M tail entries:
  the full-size tail schedule -- 8 entries per lane, up to 256-lane rows,
  the red.global.add into y): uniform x (tolerance) and the integer-exact
  regime (integer-valued matrix and x, bitwise -- pins the tail's reduction
  exactly); the degree-sorted stress variant; and the P = 8 CONTIG_NNZ
  partition through both emulated transports.

Bar (BASELINE.json north_star): |y_gpu - y_ref|_i <= 1e-12 (|A||x|)_i in fp64,
bitwise where every partial sum is an exact integer (pin P3)."""
import numpy as np
import pytest

import hecgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1606_00545_b200 as hec  # noqa: E402


def gpu_spmv(M, x):
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    yd = torch.full((M.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    M.spmv(xd, yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy()


def local_spmv(grp, pp, x):
    P = len(pp) - 1
    xs = [torch.from_numpy(np.ascontiguousarray(x[pp[p]:pp[p + 1]])).cuda() for p in range(P)]
    ys = [torch.full((int(pp[p + 1] - pp[p]),), float("nan"), dtype=torch.float64, device="cuda")
          for p in range(P)]
    grp.spmv(xs, ys)
    torch.cuda.synchronize()
    for r in grp.ranks:
        r.check()
    return np.concatenate([t.cpu().numpy() for t in ys])


def assert_all_rows(y, ref, tol, what):
    assert y.shape == ref.shape
    bad = np.nonzero(~(np.abs(y - ref) <= tol))[0]
    assert bad.size == 0, f"{what}: {bad.size} of {y.size} rows out of tolerance, first {bad[:5]}"


class Case:
    """A full-size matrix with its x vectors and oracle results (computed once)."""

    def __init__(self, A):
        self.A = A
        self.x = hecgen.vector(A.n_cols, "uniform", seed=1606)
        self.ref = oracle.csr_spmv(A, self.x)
        self.tol = oracle.tolerance(A, self.x)


@pytest.fixture(scope="module")
def p256():
    return Case(hecgen.poisson3d(256, 256, 256))


@pytest.fixture(scope="module")
def pl8m():
    return Case(hecgen.powerlaw(1 << 23))


def test_poisson_256_every_row(p256):
    A = p256.A
    M = hec.from_csr(A)
    assert (M.info.ell_width, M.info.tail_rows) == (7, 0)
    assert_all_rows(gpu_spmv(M, p256.x), p256.ref, p256.tol, "256^3 uniform x")
    y1 = gpu_spmv(M, np.ones(A.n_cols))
    assert y1.tobytes() == (6.0 - (np.diff(A.row_ptr) - 1)).astype(np.float64).tobytes()
    xi = hecgen.vector(A.n_cols, "int", seed=5)
    assert gpu_spmv(M, xi).tobytes() == oracle.csr_spmv(A, xi).tobytes()
    M.free()


@pytest.mark.parametrize("p2p", [False, True])
def test_poisson_256_8_slabs_every_row(p256, p2p):
    # the scaling run's partition; p2p: the fused push kernel + flag wait +
    # boundary rows as its programmatic dependent; two calls so both window
    # parities are used
    A = p256.A
    plan = hec.partition(A, 8, hec.PART_GRID, (256, 256, 256))
    grp = hec.LocalDistGroup(A, plan, 0, None, p2p=p2p)
    pp = plan.part_ptr()
    for _ in range(2):
        assert_all_rows(local_spmv(grp, pp, p256.x), p256.ref, p256.tol, f"256^3 / 8 slabs p2p={p2p}")
    grp.free()


def test_powerlaw_8m_every_row(pl8m):
    A = pl8m.A
    M = hec.from_csr(A)
    assert M.info.ell_width == 9 and M.info.tail_rows > 2_000_000 and M.info.tail_nnz > (1 << 22)
    assert_all_rows(gpu_spmv(M, pl8m.x), pl8m.ref, pl8m.tol, "power-law 2^23 uniform x")
    M.free()


@pytest.mark.parametrize("P", [8])
@pytest.mark.parametrize("p2p", [False, True])
def test_powerlaw_8m_contig_nnz_every_row(pl8m, P, p2p):
    A = pl8m.A
    plan = hec.partition(A, P, hec.PART_CONTIG_NNZ)
    grp = hec.LocalDistGroup(A, plan, 0, None, p2p=p2p)
    pp = plan.part_ptr()
    for _ in range(2):
        assert_all_rows(local_spmv(grp, pp, pl8m.x), pl8m.ref, pl8m.tol, f"power-law 2^23 / {P} p2p={p2p}")
    grp.free()


def test_powerlaw_8m_degree_sorted_every_row(pl8m):
    A = hecgen.degree_sorted(pl8m.A)
    x = pl8m.x
    M = hec.from_csr(A)
    assert M.info.ell_width == 9
    assert np.all(np.diff(A.row_ptr)[:M.info.tail_rows] > 9)   # the tail is exactly the top rows
    assert_all_rows(gpu_spmv(M, x), oracle.csr_spmv(A, x), oracle.tolerance(A, x), "degree-sorted 2^23")
    M.free()


def test_powerlaw_8m_integer_regime_bitwise():
    # integer-valued power-law matrix at full size (same pattern recipe) with
    # integer x: every partial sum is an exact integer < 2^53, so any order --
    # the 8-entries-per-lane schedule, the 2-8 warp rows combined through
    # shared memory, the red.global.add onto the ELL result -- must give the
    # oracle's bits on every row
    A = hecgen.powerlaw(1 << 23, integer_values=True)
    xi = hecgen.vector(A.n_cols, "int", seed=7)
    M = hec.from_csr(A)
    assert M.info.ell_width == 9 and M.info.tail_nnz > (1 << 22)
    y = gpu_spmv(M, xi)
    M.free()
    ref = oracle.csr_spmv(A, xi)
    assert np.all(np.abs(ref) < 2.0 ** 53)
    assert y.tobytes() == ref.tobytes()
