"""GPU parity of the distributed path's kernels on ONE device.

- hec_dist_create_local emulates all P ranks of a partition on one GPU: the
  same plan, sub-HECs, pack / interior / boundary kernels as hec_spmv_dist,
  with the exchange done by device-to-device copies instead of NCCL.
- hec_spmv_dist at P = 1 (one rank, no peers) runs the real NCCL-path entry
  point and must equal hec_spmv bitwise.
Multi-GPU NCCL runs need >= 2 GPUs (bench.py --gpus N under torchrun)."""
import numpy as np
import pytest

import hecgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1606_00545_b200 as hec  # noqa: E402


def run_local(A, x, P, kind, grid=None, o=None):
    plan = hec.partition(A, P, kind, grid)
    grp = hec.LocalDistGroup(A, plan, 0, o)
    pp = plan.part_ptr()
    xs = [torch.from_numpy(np.ascontiguousarray(x[pp[p]:pp[p + 1]])).cuda() for p in range(P)]
    ys = [torch.full((int(pp[p + 1] - pp[p]),), float("nan"), dtype=torch.float64, device="cuda") for p in range(P)]
    grp.spmv(xs, ys)
    torch.cuda.synchronize()
    y = np.concatenate([t.cpu().numpy() for t in ys])
    grp.free()
    return y


def assert_parity(A, x, y):
    ref = oracle.csr_spmv(A, x)
    assert np.all(np.abs(y - ref) <= oracle.tolerance(A, x))


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_local_poisson_slabs(P):
    A = hecgen.poisson3d(32, 24, 16)
    x = hecgen.vector(A.n_cols, "uniform", seed=P)
    assert_parity(A, x, run_local(A, x, P, hec.PART_GRID, (32, 24, 16)))
    xi = hecgen.vector(A.n_cols, "int", seed=P)
    assert run_local(A, xi, P, hec.PART_GRID, (32, 24, 16)).tobytes() == oracle.csr_spmv(A, xi).tobytes()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_local_powerlaw_contig_nnz(P):
    A = hecgen.powerlaw(1 << 15, seed=P)
    x = hecgen.vector(A.n_cols, "uniform", seed=P)
    assert_parity(A, x, run_local(A, x, P, hec.PART_CONTIG_NNZ))
    B = hecgen.powerlaw(1 << 14, integer_values=True, seed=P)
    xi = hecgen.vector(B.n_cols, "int", seed=P)
    assert run_local(B, xi, P, hec.PART_CONTIG_NNZ).tobytes() == oracle.csr_spmv(B, xi).tobytes()


@pytest.mark.parametrize("P", [4, 8])
def test_local_degree_sorted_contig_cost(P):
    # the §8(d) stress variant under the cost-balanced partition
    A = hecgen.degree_sorted(hecgen.powerlaw(1 << 15, seed=P))
    x = hecgen.vector(A.n_cols, "uniform", seed=P)
    assert_parity(A, x, run_local(A, x, P, hec.PART_CONTIG_COST))
    B = hecgen.degree_sorted(hecgen.powerlaw(1 << 14, integer_values=True, seed=P))
    xi = hecgen.vector(B.n_cols, "int", seed=P)
    assert run_local(B, xi, P, hec.PART_CONTIG_COST).tobytes() == oracle.csr_spmv(B, xi).tobytes()


def test_local_spe10_and_every_row_its_own_part():
    A = hecgen.spe10(20, 30, 10, seed=3)
    x = hecgen.vector(A.n_cols, "uniform", seed=3)
    assert_parity(A, x, run_local(A, x, 5, hec.PART_CONTIG_NNZ))
    B = hecgen.random_csr(24, 24, 0.2, seed=1)
    xb = hecgen.vector(24, "uniform", seed=1)
    assert_parity(B, xb, run_local(B, xb, 24, hec.PART_CONTIG_ROWS))   # P = n


def test_dist_single_rank_equals_hec_spmv_bitwise():
    A = hecgen.powerlaw(1 << 15, seed=2)
    x = torch.from_numpy(hecgen.vector(A.n_cols, "uniform", seed=2)).cuda()
    plan = hec.partition(A, 1)
    D = hec.Dist(A, plan, 0, None, 0)
    assert D.info.n_halo == 0 and D.info.n_boundary == 0
    y1 = torch.empty_like(x)
    D.spmv(x, y1)
    M = hec.from_csr(A)
    y2 = torch.empty_like(x)
    M.spmv(x, y2)
    torch.cuda.synchronize()
    assert y1.cpu().numpy().tobytes() == y2.cpu().numpy().tobytes()
    with pytest.raises(hec.HecError):
        D.phase_times()                      # no timed call yet
    D.set_timing(True)
    D.spmv(x, y1)
    t_int, t_comm = D.phase_times()
    assert t_int > 0 and t_comm == -1.0      # one rank: no exchange
    torch.cuda.synchronize()
    assert y1.cpu().numpy().tobytes() == y2.cpu().numpy().tobytes()


def test_local_group_p1_equals_hec_spmv_bitwise():
    A = hecgen.spe10(20, 30, 10, seed=7)
    x = hecgen.vector(A.n_cols, "uniform", seed=7)
    y_local = run_local(A, x, 1, hec.PART_CONTIG_NNZ)
    M = hec.from_csr(A)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    M.spmv(xd, yd)
    torch.cuda.synchronize()
    assert y_local.tobytes() == yd.cpu().numpy().tobytes()
