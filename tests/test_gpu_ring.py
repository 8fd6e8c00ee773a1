"""GPU parity of the x-ring schedule of the CSR tail (tail_ring_kernel,
DESIGN §5; Alg. 1 lines 5-7).

One CTA per SM walks a contiguous run of warp units; each stage's x window
is bulk-copied into a shared-memory ring and in-window gathers read it.  The
lanes, partial sums, reduction order and the one red.add per row are those
of the one-CTA-per-descriptor tail kernel, so every result must be BITWISE
equal to it (HEC_TAIL_RING=0), within the north_star tolerance of the
oracle, and bitwise equal to the oracle in the integer regime.  Covered:
repeated launches, rows over several warps (degree-sorted), ring-window
wrap-around, CTAs without work, the Eq. (2) / Jacobi epilogues, the halo
(distributed boundary) variant, and the fallback for a misaligned x."""
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


def dev(v):
    return torch.from_numpy(np.ascontiguousarray(v)).cuda()


def run(M, x):
    yd = torch.full((M.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    M.spmv(dev(x), yd)
    torch.cuda.synchronize()
    return yd.cpu().numpy()


def pair(A, **kv):
    """(ring handle, plain handle) of the same matrix."""
    with env(HEC_TAIL_RING=1, HEC_FUSE_TAIL=0, **kv):
        Mr = hec.from_csr(A)
    with env(HEC_TAIL_RING=0, HEC_FUSE_TAIL=0, **kv):
        Mp = hec.from_csr(A)
    assert Mr.info.tail_ring == 1 and Mp.info.tail_ring == 0
    return Mr, Mp


@pytest.mark.parametrize("n,epl", [(1 << 16, 32), (1 << 18, 32), (1 << 18, 8)])
def test_ring_bitwise_vs_plain(n, epl):
    A = hecgen.powerlaw(n, seed=21)
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    Mr, Mp = pair(A, HEC_TAIL_EPL=epl)
    # the banded power-law tail: nearly every local column is in its window
    assert Mr.info.tail_ring_cover > 0.8
    yp = run(Mp, x)
    for _ in range(3):
        assert run(Mr, x).tobytes() == yp.tobytes()
    assert np.all(np.abs(yp - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_ring_integer_bitwise_vs_oracle():
    A = hecgen.powerlaw(1 << 18, integer_values=True, seed=22)
    xi = hecgen.vector(A.n_cols, "int", seed=2)
    Mr, _ = pair(A)
    assert run(Mr, xi).tobytes() == oracle.csr_spmv(A, xi).tobytes()


def test_ring_long_rows_degree_sorted():
    # rows of up to 2,000 entries (G = 64-256 lanes: one warp walks the row's
    # G/32 warp chunks) and a window that covers few columns
    A = hecgen.degree_sorted(hecgen.powerlaw(1 << 17, seed=23))
    x = hecgen.vector(A.n_cols, "uniform", seed=3)
    Mr, Mp = pair(A)
    assert run(Mr, x).tobytes() == run(Mp, x).tobytes()


def test_ring_small_matrix_idle_ctas():
    # fewer warp units than SMs: most CTAs have no stage
    A = hecgen.powerlaw(1 << 11, seed=24)
    x = hecgen.vector(A.n_cols, "uniform", seed=4)
    Mr, Mp = pair(A)
    assert run(Mr, x).tobytes() == run(Mp, x).tobytes()


def test_ring_epilogues_bitwise():
    A = hecgen.powerlaw(1 << 17, seed=25)
    n = A.n_rows
    x = hecgen.vector(n, "uniform", seed=5)
    y0 = hecgen.vector(n, "uniform", seed=6)
    Mr, Mp = pair(A)
    outs = []
    for M in (Mr, Mp):
        y = dev(y0)
        M.spmv_axpby(-0.75, dev(x), 0.5, y)  # Eq. (2)
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        M.diag(d)
        xo = torch.empty(n, dtype=torch.float64, device="cuda")
        M.jacobi(d, dev(y0), dev(x), xo, 0.8)  # damped Jacobi (A22)
        torch.cuda.synchronize()
        outs.append((y.cpu().numpy().tobytes(), xo.cpu().numpy().tobytes()))
    assert outs[0] == outs[1]


def test_ring_misaligned_x_falls_back():
    # x not 16-byte aligned: the bulk copies cannot run, the plain tail kernel does
    A = hecgen.powerlaw(1 << 16, seed=26)
    x = hecgen.vector(A.n_cols, "uniform", seed=7)
    Mr, Mp = pair(A)
    buf = torch.empty(A.n_cols + 1, dtype=torch.float64, device="cuda")
    buf[1:] = dev(x)
    y = torch.full((A.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    Mr.spmv(buf[1:], y)
    torch.cuda.synchronize()
    assert y.cpu().numpy().tobytes() == run(Mp, x).tobytes()


@pytest.mark.parametrize("P", [2, 4])
def test_ring_distributed_halo(P):
    # interior and boundary sub-HECs (local columns in the ring, halo columns
    # from x_halo), all parts on this GPU
    A = hecgen.powerlaw(1 << 17, seed=27)
    x = hecgen.vector(A.n_cols, "uniform", seed=8)
    plan = hec.partition(A, P, hec.PART_CONTIG_NNZ)
    pp = plan.part_ptr()
    ys = {}
    for ring in (1, 0):
        with env(HEC_TAIL_RING=ring):
            grp = hec.LocalDistGroup(A, plan, 0, None, p2p=True)
        xs = [dev(x[pp[p]:pp[p + 1]]) for p in range(P)]
        yl = [torch.full((int(pp[p + 1] - pp[p]),), float("nan"), dtype=torch.float64, device="cuda")
              for p in range(P)]
        grp.spmv(xs, yl)
        torch.cuda.synchronize()
        ys[ring] = np.concatenate([t.cpu().numpy() for t in yl])
        grp.free()
    assert ys[1].tobytes() == ys[0].tobytes()
    assert np.all(np.abs(ys[1] - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_ring_full_size_powerlaw_every_row():
    # configs[4] (2^23 rows, 79 M tail entries): every row bitwise equal to
    # the plain schedule (the ring is opt-in: slower there)
    A = hecgen.powerlaw(1 << 23, seed=1)
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    with env(HEC_TAIL_RING=1, HEC_FUSE_TAIL=0):
        Mr = hec.from_csr(A)
    assert Mr.info.tail_ring == 1 and Mr.info.tail_ring_cover > 0.85
    yr = run(Mr, x)
    Mr.free()
    Mp = hec.from_csr(A)
    assert Mp.info.tail_ring == 0
    assert yr.tobytes() == run(Mp, x).tobytes()
