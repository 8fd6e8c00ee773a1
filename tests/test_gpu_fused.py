"""GPU parity of the small-tail "tail first" path: for a whole matrix whose CSR
tail kernel fits one wave, hec_spmv runs Alg. 1 lines 5-7 FIRST,
storing each tail row's sum into y, and the ELL kernel (lines 1-3), launched
as its programmatic dependent, adds the stored sums in the CTAs that own tail
rows.  Same lanes, order and single rounding y_i = ell_i + tail_i as the
ELL-then-tail path, so the two products must be BITWISE equal; both within the
north_star tolerance of the oracle (bitwise on integer data).
HEC_FUSE_TAIL=0 forces the ELL-then-tail order."""
import os

import numpy as np
import pytest

import hecgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1606_00545_b200 as hec  # noqa: E402


def build(A, fuse: bool, o=None):
    old = os.environ.get("HEC_FUSE_TAIL")
    os.environ["HEC_FUSE_TAIL"] = "1" if fuse else "0"
    try:
        return hec.from_csr(A, o)
    finally:
        if old is None:
            os.environ.pop("HEC_FUSE_TAIL", None)
        else:
            os.environ["HEC_FUSE_TAIL"] = old


def run(M, x):
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    yd = torch.full((M.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    M.spmv(xd, yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy()


def long_rows():
    rows = [[], [(0, 1.0)], [(c, 1.0) for c in range(5)], [(c, -2.0) for c in range(6)], [],
            [(c, 0.5 + c % 3) for c in range(4000)], [], [(c, 0.25 * (c % 5) - 0.5) for c in range(0, 4000, 37)]]
    return hecgen.from_rows(4000, rows)


CASES = [
    ("spe10_full", lambda: hecgen.spe10(60, 220, 85), None),                  # configs[3]: 78 tail rows, wells
    ("spe10_small", lambda: hecgen.spe10(20, 30, 10, seed=5), None),
    ("long_rows_256_lanes", long_rows, None),                                  # a 4,000-entry row: 8 virtual warps
    ("powerlaw_4k", lambda: hecgen.powerlaw(4096, seed=2), None),
    ("powerlaw_4k_cap20", lambda: hecgen.powerlaw(4096, seed=3), hec.opts(hec.WIDTH_CAP, 20)),
    ("random_rect", lambda: hecgen.random_csr(3000, 700, 0.02, seed=4), hec.opts(hec.WIDTH_FIXED, 0, 3)),
]


@pytest.mark.parametrize("name,maker,o", CASES)
def test_fused_equals_two_kernel_bitwise_and_oracle(name, maker, o):
    A = maker()
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    Mf, M2 = build(A, True, o), build(A, False, o)
    assert M2.info.tail_rows > 0 and M2.launches == 2 and M2.info.tail_fused == 0
    assert Mf.info.tail_fused == 1, name           # tail first, ELL as its dependent
    yf, y2 = run(Mf, x), run(M2, x)
    assert yf.tobytes() == y2.tobytes()
    assert np.all(np.abs(yf - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_fused_integer_bitwise():
    A = hecgen.powerlaw(8192, integer_values=True, seed=5)
    xi = hecgen.vector(A.n_cols, "int", seed=1)
    M = build(A, True)
    assert M.info.tail_fused == 1
    assert run(M, xi).tobytes() == oracle.csr_spmv(A, xi).tobytes()


def test_fused_all_rows_in_the_tail():
    # CAP 0: width 0, every row is a tail row: the ELL kernel only adds the
    # stored sums (every CTA waits for the tail grid)
    A = hecgen.powerlaw(3000, seed=6)
    Mf, M2 = build(A, True, hec.opts(hec.WIDTH_CAP, 0)), build(A, False, hec.opts(hec.WIDTH_CAP, 0))
    assert Mf.info.ell_width == 0 and Mf.info.tail_fused == 1
    x = hecgen.vector(A.n_cols, "uniform", seed=2)
    yf = run(Mf, x)
    assert yf.tobytes() == run(M2, x).tobytes()
    assert np.all(np.abs(yf - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_fused_epilogues_and_host_path_use_two_kernels_consistently():
    # axpby / Jacobi / hec_spmv_host keep the two-kernel path on a fused
    # handle; y = 1 * A x + 0 * y through axpby equals the fused product
    A = hecgen.spe10(20, 30, 10, seed=9)
    x = hecgen.vector(A.n_cols, "uniform", seed=3)
    M = build(A, True)
    assert M.info.tail_fused == 1
    y = run(M, x)
    yd = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
    M.spmv_axpby(2.0, torch.from_numpy(x).cuda(), 0.0, yd)
    torch.cuda.synchronize()
    assert np.all(np.abs(yd.cpu().numpy() - 2.0 * oracle.csr_spmv(A, x)) <= 2 * oracle.tolerance(A, x))
    assert M.spmv_host(x).tobytes() == y.tobytes()
