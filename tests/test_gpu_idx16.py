"""GPU parity of the ELL index compression (Alg. 1 lines 1-3,
P:132-134): slot j of row i streams the int16 delta col - i - base_j instead
of the int32 column (padding and deltas that do not fit take the escape
codes; an escaped slot reads its int32 column).  The decoded column equals
the stored one, so every product must be BITWISE equal to the uncompressed
path (HEC_IDX16=0) and within the north_star tolerance of the oracle
(bitwise in the integer regime).  The compression is opt-in (HEC_IDX16=1;
measured no faster).  Covered: stencils and reservoir matrices
(few escapes), matrices full of escapes and padding, odd row counts, the
chunked host path (row offsets), the Eq. (2) and Jacobi epilogues and the
distributed sub-matrices (row maps and halo columns)."""
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


def pair(A):
    with env(HEC_IDX16=1):
        Mc = hec.from_csr(A)
    Mp = hec.from_csr(A)  # the default: int32 columns
    assert Mc.info.ell_idx16 == 1 and Mp.info.ell_idx16 == 0
    return Mc, Mp


@pytest.mark.parametrize("maker", [lambda: hecgen.poisson3d(40, 30, 50), lambda: hecgen.poisson2d(64, 64),
                                   lambda: hecgen.poisson3d(17, 5, 3), lambda: hecgen.spe10(20, 30, 10, seed=3)])
def test_idx16_stencils_bitwise(maker):
    A = maker()
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    Mc, Mp = pair(A)
    assert Mc.info.ell_idx16 == 1 and 0.0 <= Mc.info.ell_idx16_escaped <= 0.02
    yc = run(Mc, x)
    assert yc.tobytes() == run(Mp, x).tobytes()
    assert np.all(np.abs(yc - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_idx16_integer_regime_bitwise_vs_oracle():
    A = hecgen.poisson3d(33, 20, 31)
    xi = hecgen.vector(A.n_cols, "int", seed=2)
    Mc, _ = pair(A)
    assert run(Mc, xi).tobytes() == oracle.csr_spmv(A, xi).tobytes()


def test_idx16_powerlaw_escapes_reported():
    # far columns escape; the fraction is reported (and -1 when not evaluated)
    A = hecgen.powerlaw(1 << 16, seed=3)
    Mc, Mp = pair(A)
    assert Mc.info.ell_idx16_escaped > 0.02 and Mp.info.ell_idx16_escaped == -1.0


@pytest.mark.parametrize("maker", [lambda: hecgen.powerlaw(1 << 16, seed=3),
                                   lambda: hecgen.random_csr(5001, 200_000, 0.00004, seed=4),
                                   lambda: hecgen.degree_sorted(hecgen.powerlaw(1 << 15, seed=5))])
def test_idx16_forced_escapes_bitwise(maker):
    A = maker()
    x = hecgen.vector(A.n_cols, "uniform", seed=7)
    Mc, Mp = pair(A)
    assert Mc.info.ell_idx16 == 1
    yc = run(Mc, x)
    assert yc.tobytes() == run(Mp, x).tobytes()
    assert np.all(np.abs(yc - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_idx16_host_chunks_bitwise():
    # >= 2M rows: hec_spmv_host's row chunks (each launch starts at a row offset)
    A = hecgen.poisson3d(128, 128, 130)
    x = hecgen.vector(A.n_cols, "uniform", seed=4)
    Mc, Mp = pair(A)
    assert Mc.info.ell_idx16 == 1
    yp = run(Mp, x)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.full((A.n_rows,), float("nan"), dtype=torch.float64).pin_memory()
    Mc.spmv_host(xh, yh)
    assert yh.numpy().tobytes() == yp.tobytes()
    assert run(Mc, x).tobytes() == yp.tobytes()


def test_idx16_epilogues_bitwise():
    A = hecgen.poisson3d(30, 31, 32)
    n = A.n_rows
    x = hecgen.vector(n, "uniform", seed=5)
    y0 = hecgen.vector(n, "uniform", seed=6)
    Mc, Mp = pair(A)
    outs = []
    for M in (Mc, Mp):
        y = dev(y0)
        M.spmv_axpby(-0.75, dev(x), 0.5, y)  # Eq. (2)
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        M.diag(d)
        xo = torch.empty(n, dtype=torch.float64, device="cuda")
        M.jacobi(d, dev(y0), dev(x), xo, 0.8)  # damped Jacobi (A22)
        torch.cuda.synchronize()
        outs.append((y.cpu().numpy().tobytes(), xo.cpu().numpy().tobytes()))
    assert outs[0] == outs[1]


@pytest.mark.parametrize("P", [2, 4])
def test_idx16_distributed_bitwise(P):
    # interior (row map) and boundary (halo columns, mostly escapes) sub-HECs
    A = hecgen.poisson3d(24, 24, 32)
    x = hecgen.vector(A.n_cols, "uniform", seed=8)
    plan = hec.partition(A, P, hec.PART_GRID, grid=(24, 24, 32))
    pp = plan.part_ptr()
    ys = {}
    for flag in (1, 0):
        with env(HEC_IDX16=flag):
            grp = hec.LocalDistGroup(A, plan, 0, None, p2p=True)
        xs = [dev(x[pp[p]:pp[p + 1]]) for p in range(P)]
        yl = [torch.full((int(pp[p + 1] - pp[p]),), float("nan"), dtype=torch.float64, device="cuda")
              for p in range(P)]
        grp.spmv(xs, yl)
        torch.cuda.synchronize()
        ys[flag] = np.concatenate([t.cpu().numpy() for t in yl])
        grp.free()
    assert ys[1].tobytes() == ys[0].tobytes()
    assert np.all(np.abs(ys[1] - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_idx16_full_size_poisson_256_every_row():
    # the bench workload (configs[2]) compressed: every row bitwise equal to
    # the int32 path
    A = hecgen.poisson3d(256, 256, 256)
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    with env(HEC_IDX16=1):
        M = hec.from_csr(A)
    assert M.info.ell_idx16 == 1 and M.info.ell_idx16_escaped < 0.01
    yc = run(M, x)
    M.free()
    Mp = hec.from_csr(A)
    assert yc.tobytes() == run(Mp, x).tobytes()
