"""CSR -> HEC conversion (libhec host converter) vs the oracle builder O2,
BIT-EXACT (BASELINE.json north_star: "the HEC conversion ... must match
bit-exactly").  Host-only handles (device = -1), so this runs without a GPU."""
import numpy as np
import pytest

import hecgen
import paper_1606_00545_b200 as hec
from oracle import hec_ref as H


def assert_same(A, o, ref):
    M = hec.from_csr(A, o, device=-1)
    got = M.export()
    assert (got.width, got.stride) == (ref.width, ref.stride)
    assert M.info.nnz == A.nnz and M.info.ell_nnz + M.info.tail_nnz == A.nnz
    for f in ("ell_col", "ell_val", "tail_rows", "tail_ptr", "tail_col", "tail_val"):
        a, b = getattr(got, f), getattr(ref, f)
        assert a.dtype == b.dtype and a.shape == b.shape, f
        assert a.tobytes() == b.tobytes(), f          # bitwise (incl. +0.0 padding)
    return M


POLICIES = [(hec.WIDTH_BG3, 20, 0), (hec.WIDTH_BG3, 3, 0), (hec.WIDTH_CAP, 20, 0), (hec.WIDTH_CAP, 0, 0),
            (hec.WIDTH_FIXED, 0, 4), (hec.WIDTH_FIXED, 0, 0)]


@pytest.mark.parametrize("policy,cap,fixed", POLICIES)
@pytest.mark.parametrize("unit", [32, 256])
def test_random_small_bitexact(policy, cap, fixed, unit):
    for seed, (n, m, d) in enumerate([(1, 1, 1.0), (31, 31, 0.2), (32, 40, 0.3), (33, 20, 0.5), (255, 64, 0.05),
                                      (256, 256, 0.02), (257, 100, 0.1), (5, 3, 0.8), (3, 5, 0.8), (10, 10, 0.0)]):
        A = hecgen.random_csr(n, m, d, seed=500 + seed)
        o = hec.opts(policy, cap, fixed, unit)
        assert_same(A, o, H.build_fast(A, policy, cap, fixed, unit))


def test_spec_examples():
    assert_same(hecgen.from_dense(np.eye(4)), hec.opts(hec.WIDTH_CAP, 20, 0, 32),
                H.build(hecgen.from_dense(np.eye(4)), H.POLICY_CAP, 20, 0, 32))
    rows = [[(0, 1.0), (1, 2.0)], [(1, 3.0), (2, 4.0)], [(2, 5.0), (3, 6.0)], [(c, c + 1.0) for c in range(25)]]
    A = hecgen.from_rows(25, rows)
    M = assert_same(A, hec.opts(hec.WIDTH_CAP, 20, 0, 32), H.build(A, H.POLICY_CAP, 20, 0, 32))
    assert M.info.ell_width == 20 and M.info.tail_nnz == 5
    M = assert_same(A, hec.opts(hec.WIDTH_CAP, 0, 0, 32), H.build(A, H.POLICY_CAP, 0, 0, 32))
    assert M.info.ell_width == 0 and M.info.tail_nnz == A.nnz


def test_edge_rows():
    # empty rows, a row of exactly w, w+1 (one tail entry), a 4000-entry row
    rows = [[], [(0, 1.0)], [(c, 1.0) for c in range(5)], [(c, 2.0) for c in range(6)], [],
            [(c, 0.5) for c in range(4000)]]
    rows += [[(i % 4000, 1.0), ((i * 7) % 4000 + 0, 1.0)] if (i * 7) % 4000 > i % 4000 else [(i % 4000, 1.0)]
             for i in range(200)]
    A = hecgen.from_rows(4000, rows)
    for o, args in [(hec.opts(hec.WIDTH_FIXED, 0, 5), (H.POLICY_FIXED, 0, 5)), (hec.opts(), (H.POLICY_BG3, 20, 0))]:
        assert_same(A, o, H.build(A, *args))


def test_empty_matrix():
    A = hecgen.from_dense(np.zeros((0, 0)))
    M = assert_same(A, hec.opts(), H.build(A))
    assert M.info.n_rows == 0 and M.info.ell_stride == 0
    Z = hecgen.from_dense(np.zeros((7, 3)))
    assert_same(Z, hec.opts(), H.build(Z))


@pytest.mark.parametrize("maker", [lambda: hecgen.poisson2d(64, 64), lambda: hecgen.poisson3d(32, 32, 32),
                                   lambda: hecgen.spe10(60, 220, 85), lambda: hecgen.powerlaw(1 << 17),
                                   lambda: hecgen.powerlaw(20000, integer_values=True, seed=9)])
def test_workload_shapes_bitexact(maker):
    A = maker()
    M = assert_same(A, hec.opts(), H.build_fast(A))
    if A.name.startswith("poisson2d_64"):
        assert (M.info.ell_width, M.info.tail_rows) == (5, 0)
    if A.name.startswith("spe10"):
        # 5 well rows + the perforated cells (8 entries) spill at w = 7
        assert M.info.ell_width == 7 and 70 <= M.info.tail_rows <= 90


def test_poisson_128_bitexact():
    A = hecgen.poisson3d(128, 128, 128)
    M = assert_same(A, hec.opts(), H.build_fast(A))
    assert (M.info.ell_width, M.info.ell_stride, M.info.tail_rows) == (7, 128 ** 3, 0)
