"""GPU parity of the CSR-tail kernel (Alg. 1 lines 5-7) in its
warp-chunk device layout (hec_internal.h) under every lanes-per-row regime
the planner can pick: HEC_TAIL_EPL (target entries per lane) moves rows
between G = 1 lane (many rows per warp) and G = 256 lanes (a row over 8
warps), which changes which rows share a warp, how much padding the layout
carries and how many batched iterations a lane runs.  Every setting must
match the oracle within the north_star tolerance, bitwise on integer data,
and hec_export must give back the host CSR tail exactly."""
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


class env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run(M, x):
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    yd = torch.full((M.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    M.spmv(xd, yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy()


@pytest.mark.parametrize("epl", [1, 2, 8, 32, 64])
def test_tail_every_lane_regime(epl):
    A = hecgen.powerlaw(1 << 16, seed=3)
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    with env(HEC_TAIL_EPL=epl, HEC_FUSE_TAIL=0):
        M = hec.from_csr(A)
    assert M.launches == 2
    y = run(M, x)
    assert np.all(np.abs(y - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))
    e, r = M.export(), hec.from_csr(A, device=-1).export()
    for f in ("tail_rows", "tail_ptr", "tail_col", "tail_val"):
        assert getattr(e, f).tobytes() == getattr(r, f).tobytes()


@pytest.mark.parametrize("epl", [2, 32])
def test_tail_integer_bitwise(epl):
    A = hecgen.powerlaw(1 << 16, integer_values=True, seed=6)
    xi = hecgen.vector(A.n_cols, "int", seed=2)
    with env(HEC_TAIL_EPL=epl, HEC_FUSE_TAIL=0):
        M = hec.from_csr(A)
    assert run(M, xi).tobytes() == oracle.csr_spmv(A, xi).tobytes()


def test_tail_degree_sorted_long_rows_first():
    # the longest rows (2,000 entries: 64-256 lanes over 2-8 warps) all in the
    # first super-blocks
    A = hecgen.degree_sorted(hecgen.powerlaw(1 << 16, seed=7))
    x = hecgen.vector(A.n_cols, "uniform", seed=3)
    for epl in (8, 32):
        with env(HEC_TAIL_EPL=epl, HEC_FUSE_TAIL=0):
            M = hec.from_csr(A)
        assert np.all(np.abs(run(M, x) - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


@pytest.mark.parametrize("P", [2, 4])
def test_tail_distributed_halo_regimes(P):
    # boundary sub-HECs: the halo tail kernel (fewer batched iterations)
    A = hecgen.powerlaw(1 << 16, seed=8)
    x = hecgen.vector(A.n_cols, "uniform", seed=8)
    plan = hec.partition(A, P, hec.PART_CONTIG_NNZ)
    pp = plan.part_ptr()
    for epl in (2, 32):
        with env(HEC_TAIL_EPL=epl):
            grp = hec.LocalDistGroup(A, plan, 0, None, p2p=True)
        xs = [torch.from_numpy(np.ascontiguousarray(x[pp[p]:pp[p + 1]])).cuda() for p in range(P)]
        ys = [torch.full((int(pp[p + 1] - pp[p]),), float("nan"), dtype=torch.float64, device="cuda")
              for p in range(P)]
        grp.spmv(xs, ys)
        torch.cuda.synchronize()
        y = np.concatenate([t.cpu().numpy() for t in ys])
        grp.free()
        assert np.all(np.abs(y - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_tail_jacobi_diag_regimes():
    A = hecgen.powerlaw(1 << 15, seed=9)
    for epl in (2, 32):
        with env(HEC_TAIL_EPL=epl, HEC_FUSE_TAIL=0):
            M = hec.from_csr(A)
        d = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
        M.diag(d)
        torch.cuda.synchronize()
        ref = np.array([A.val[k] for i in range(A.n_rows) for k in range(A.row_ptr[i], A.row_ptr[i + 1])
                        if A.col[k] == i])
        assert d.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("integer", [False, True])
def test_tail_sm_local_warp_schedule_bitwise(integer):
    # the SM-local persistent schedule, warp by warp (whole launches of tails
    # with more descriptors than one wave): the same warp chunks, partial sums
    # and reduction order -- bitwise equal to the one-CTA-per-descriptor grid,
    # over repeated launches (the claim counters reset themselves)
    A = hecgen.powerlaw(1 << 18, integer_values=integer, seed=11)
    if not integer:  # long rows (G > 32: one warp walks the row's G/32 warp chunks)
        A = hecgen.degree_sorted(A)
    x = hecgen.vector(A.n_cols, "int" if integer else "uniform", seed=4)
    with env(HEC_TAIL_WARP=1, HEC_FUSE_TAIL=0):
        Ms = hec.from_csr(A)
    with env(HEC_TAIL_WARP=0, HEC_FUSE_TAIL=0):
        Mp = hec.from_csr(A)
    ys = [run(Ms, x) for _ in range(3)]
    yp = run(Mp, x)
    assert all(y.tobytes() == yp.tobytes() for y in ys)
    if integer:
        assert yp.tobytes() == oracle.csr_spmv(A, x).tobytes()
    else:
        assert np.all(np.abs(yp - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_tail_concurrent_stream_bitwise():
    # HEC_TAIL_CONC=1: the tail kernel on its own stream beside the ELL kernel,
    # sums into a scratch, one combine pass -- bitwise the ELL-then-tail y
    A = hecgen.powerlaw(1 << 18, seed=12)
    x = hecgen.vector(A.n_cols, "uniform", seed=5)
    with env(HEC_TAIL_CONC=1, HEC_FUSE_TAIL=0):
        Mc = hec.from_csr(A)
    with env(HEC_TAIL_CONC=0, HEC_FUSE_TAIL=0):
        Mp = hec.from_csr(A)
    yp = run(Mp, x)
    for _ in range(3):
        assert run(Mc, x).tobytes() == yp.tobytes()


@pytest.mark.parametrize("integer", [False, True])
def test_tail_reverse_descriptor_order_bitwise(integer):
    # the tail launch may walk its descriptors last to first (the default for
    # tails without heavy leading descriptors): every row still gets exactly
    # one red.add of the same sum -- bitwise equal to the forward order
    A = hecgen.powerlaw(1 << 18, integer_values=integer, seed=13)
    x = hecgen.vector(A.n_cols, "int" if integer else "uniform", seed=6)
    ys = []
    for rev in (0, 1):
        with env(HEC_TAIL_REVERSE=rev, HEC_FUSE_TAIL=0):
            M = hec.from_csr(A)
        ys.append(run(M, x))
    assert ys[0].tobytes() == ys[1].tobytes()
    if integer:
        assert ys[0].tobytes() == oracle.csr_spmv(A, x).tobytes()
