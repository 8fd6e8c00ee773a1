"""GPU parity of hec_spmv (ELL kernel + CSR-tail kernel, sm_100a) against the
serial CPU oracle O1, called through the C ABI.

Bar (BASELINE.json north_star): |y_gpu - y_ref|_i <= 1e-12 (|A||x|)_i in fp64;
bitwise in the integer-exact regime (pin P3: every partial sum is an exact
integer, so any summation order gives the same bits)."""
import numpy as np
import pytest

import hecgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1606_00545_b200 as hec  # noqa: E402


def gpu_spmv(A, x, o=None, M=None):
    M = M or hec.from_csr(A, o)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    yd = torch.full((A.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    M.spmv(xd, yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy(), M


def assert_parity(A, x, y, r0=0, r1=None):
    ref = oracle.csr_spmv(A, x, r0, r1)
    tol = oracle.tolerance(A, x, r0, r1)
    bad = np.nonzero(~(np.abs(y - ref) <= tol))[0]
    assert bad.size == 0, f"{bad.size} rows out of tolerance, first {bad[:5]}: {y[bad[:5]]} vs {ref[bad[:5]]}"


CONFIGS = [
    ("poisson2d_64", lambda: hecgen.poisson2d(64, 64)),          # BASELINE configs[0]
    ("poisson3d_32", lambda: hecgen.poisson3d(32, 32, 32)),
    ("spe10", lambda: hecgen.spe10(60, 220, 85)),                # configs[3], full size
    ("powerlaw_64k", lambda: hecgen.powerlaw(1 << 16)),
    ("powerlaw_64k_dsorted", lambda: hecgen.degree_sorted(hecgen.powerlaw(1 << 16))),  # §8(d) stress variant
    ("random_rect", lambda: hecgen.random_csr(300, 170, 0.05, seed=3)),
]


@pytest.mark.parametrize("name,maker", CONFIGS)
def test_parity_uniform_x(name, maker):
    A = maker()
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    y, M = gpu_spmv(A, x)
    assert_parity(A, x, y)
    if name == "spe10":
        assert M.info.tail_rows > 0 and M.launches == 2        # the CSR tail is exercised (tail first: M.info.tail_fused)


@pytest.mark.parametrize("name,maker", CONFIGS[:5])
def test_integer_regime_bitwise(name, maker):
    A = maker()
    if name == "spe10":
        pytest.skip("SPE10 coefficients are not integers")
    if name.startswith("powerlaw"):
        A = hecgen.powerlaw(1 << 16, integer_values=True)
        if name.endswith("dsorted"):
            A = hecgen.degree_sorted(A)
    x = hecgen.vector(A.n_cols, "int", seed=7)
    y, _ = gpu_spmv(A, x)
    assert y.tobytes() == oracle.csr_spmv(A, x).tobytes()


def test_poisson_128_full_parity():
    # BASELINE configs[1] at full size, element by element.
    A = hecgen.poisson3d(128, 128, 128)
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    y, M = gpu_spmv(A, x)
    assert (M.info.ell_width, M.info.tail_rows) == (7, 0)
    assert_parity(A, x, y)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 255, 256, 257, 1023])
@pytest.mark.parametrize("unit", [32, 256])
def test_sizes_and_strides(n, unit):
    A = hecgen.random_csr(n, n, min(1.0, 6.0 / n), seed=n)
    x = hecgen.vector(n, "uniform", seed=n)
    y, M = gpu_spmv(A, x, hec.opts(stride_unit=unit))
    assert M.info.ell_stride % unit == 0
    assert_parity(A, x, y)


def test_edge_rows_and_long_tail_row():
    rows = [[], [(0, 1.0)], [(c, 1.0) for c in range(5)], [(c, -2.0) for c in range(6)], [],
            [(c, 0.5 + c % 3) for c in range(4000)], []]
    A = hecgen.from_rows(4000, rows)
    x = hecgen.vector(4000, "uniform", seed=2)
    for o in (hec.opts(), hec.opts(hec.WIDTH_FIXED, 0, 5), hec.opts(hec.WIDTH_CAP, 0), hec.opts(hec.WIDTH_CAP, 20)):
        y, M = gpu_spmv(A, x, o)
        assert_parity(A, x, y)
        assert y[0] == 0.0 and y[4] == 0.0 and y[6] == 0.0      # empty rows -> +0.0 (A6)


def test_cap_zero_all_tail_and_no_tail():
    A = hecgen.powerlaw(5000, seed=4)
    x = hecgen.vector(A.n_cols, "uniform", seed=4)
    for o in (hec.opts(hec.WIDTH_CAP, 0), hec.opts(hec.WIDTH_CAP, 2000)):
        y, M = gpu_spmv(A, x, o)
        assert_parity(A, x, y)
    assert M.info.tail_rows == 0


@pytest.mark.parametrize("shape", [(5, 3), (3, 5), (1000, 10), (10, 1000)])
def test_rectangular(shape):
    A = hecgen.random_csr(shape[0], shape[1], 0.4, integer_values=True, seed=sum(shape))
    x = hecgen.vector(shape[1], "int", seed=1)
    y, _ = gpu_spmv(A, x)
    assert y.tobytes() == oracle.csr_spmv(A, x).tobytes()


def test_padding_and_unreachable_inf():
    # Reading A4: padding is (-1, +0.0) and the kernel predicates the x load and
    # the FMA on col >= 0, so x entries no stored entry references may be Inf/NaN.
    R = hecgen.random_csr(200, 100, 0.06, seed=8)
    A = hecgen.Csr(200, 200, R.row_ptr, (2 * R.col).astype(np.int32), R.val)   # only even columns stored
    used = np.zeros(200, bool)
    used[A.col] = True
    x = hecgen.vector(200, "uniform", seed=3)
    x[~used] = np.inf
    assert (~used).sum() >= 100
    for o in (hec.opts(hec.WIDTH_CAP, 20), hec.opts(), hec.opts(hec.WIDTH_FIXED, 0, 3)):
        y, M = gpu_spmv(A, x, o)
        assert np.all(np.isfinite(y))
        assert_parity(A, x, y)


def test_empty_matrix_and_zero_rows():
    A = hecgen.from_dense(np.zeros((6, 4)))
    y, _ = gpu_spmv(A, np.ones(4))
    assert y.tolist() == [0.0] * 6


def test_spmv_host_matches_device():
    A = hecgen.spe10(20, 30, 10, seed=5)
    x = hecgen.vector(A.n_cols, "uniform", seed=9)
    M = hec.from_csr(A)
    yd, _ = gpu_spmv(A, x, M=M)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.empty(A.n_rows, dtype=torch.float64).pin_memory()
    M.spmv_host(xp, yp)
    assert yp.numpy().tobytes() == yd.tobytes()
    yn = M.spmv_host(x)
    assert yn.tobytes() == yd.tobytes()


@pytest.mark.parametrize("maker", [lambda: hecgen.poisson3d(128, 128, 160),
                                   lambda: hecgen.powerlaw(3 << 20, seed=6),
                                   lambda: hecgen.random_csr(2_200_000, 40, 0.1, seed=2)])
def test_spmv_host_pipelined_chunks_bitwise(maker):
    # >= 2M rows: hec_spmv_host splits rows into chunks that start as soon as
    # their x prefix has arrived; the result must equal hec_spmv bit for bit.
    A = maker()
    x = hecgen.vector(A.n_cols, "uniform", seed=4)
    M = hec.from_csr(A)
    yd, _ = gpu_spmv(A, x, M=M)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.full((A.n_rows,), float("nan"), dtype=torch.float64).pin_memory()
    for _ in range(2):                       # reuse of the staging buffers and events
        M.spmv_host(xp, yp)
        assert yp.numpy().tobytes() == yd.tobytes()
    r0 = A.n_rows // 2
    assert_parity(A, x, yp.numpy()[r0:r0 + 3000], r0, r0 + 3000)


def test_export_from_device_matches_host_handle():
    A = hecgen.powerlaw(3000, seed=12)
    Md = hec.from_csr(A)
    Mh = hec.from_csr(A, device=-1)
    a, b = Md.export(), Mh.export()
    for f in ("ell_col", "ell_val", "tail_rows", "tail_ptr", "tail_col", "tail_val"):
        assert getattr(a, f).tobytes() == getattr(b, f).tobytes()


def test_aliasing_rejected_and_stream_order():
    A = hecgen.poisson2d(16, 16)
    M = hec.from_csr(A)
    buf = torch.zeros(256, dtype=torch.float64, device="cuda")
    with pytest.raises(hec.HecError) as e:
        M.spmv(buf, buf)
    assert e.value.status == 1
    # async on a user stream, ordered with torch work on that stream
    s = torch.cuda.Stream()
    x = torch.ones(256, dtype=torch.float64, device="cuda")
    y = torch.empty(256, dtype=torch.float64, device="cuda")
    with torch.cuda.stream(s):
        x.mul_(2.0)
        M.spmv(x, y, stream=s)
        y.add_(1.0)
    s.synchronize()
    ref = oracle.csr_spmv(A, 2.0 * np.ones(256)) + 1.0
    assert y.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("maker", [lambda: hecgen.powerlaw(1 << 16, seed=8), lambda: hecgen.spe10(60, 220, 85),
                                   lambda: hecgen.random_csr(500, 300, 0.05, seed=4)])
def test_hyb_comparison_variant_parity(maker):
    # NEXT-2: ELL + COO remainder (Bell-Garland HYB).  Atomic order is not fixed:
    # parity within tolerance; bitwise only on integer data.
    A = maker()
    x = hecgen.vector(A.n_cols, "uniform", seed=5)
    M = hec.from_csr_hyb(A)
    y, _ = gpu_spmv(A, x, M=M)
    assert_parity(A, x, y)
    e, r = M.export(), hec.from_csr(A, device=-1).export()
    for f in ("ell_col", "ell_val", "tail_rows", "tail_ptr", "tail_col", "tail_val"):
        assert getattr(e, f).tobytes() == getattr(r, f).tobytes()


def test_hyb_integer_bitwise_and_axpby():
    A = hecgen.powerlaw(1 << 15, integer_values=True, seed=9)
    x = hecgen.vector(A.n_cols, "int", seed=3)
    M = hec.from_csr_hyb(A)
    y, _ = gpu_spmv(A, x, M=M)
    assert y.tobytes() == oracle.csr_spmv(A, x).tobytes()
    y0 = hecgen.vector(A.n_rows, "int", seed=4)
    yd = torch.from_numpy(y0.copy()).cuda()
    M.spmv_axpby(2.0, torch.from_numpy(x).cuda(), -1.0, yd)
    torch.cuda.synchronize()
    assert yd.cpu().numpy().tobytes() == (2.0 * oracle.csr_spmv(A, x) - y0).tobytes()
