"""GPU parity of the ELL second-phase slot skipping (EllArgs::tile_w, DESIGN
§5; Alg. 1 lines 1-3): for two-phase widths the kernel reads the
second phase's slots only up to the longest ELL row of each warp's 64 rows.
The skipped slots are padding for every row of the tile and add exactly what
padding adds, so every result must be BITWISE equal to the full read
(HEC_TILE_SKIP=0), within the north_star tolerance of the oracle and bitwise
equal to it in the integer regime.  Covered: the default choice (on for
degree-sorted rows, off for the natural power-law), forced skipping, the
Eq. (2) and Jacobi epilogues, the chunked host path (row offsets) and the
distributed sub-matrices (row maps, halo columns); and the grouping of ELL
rows by length inside 1024-row windows that makes the natural power-law's
slots skippable (y through the permutation, hec_export back in row order)."""
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


def pair(A, force=False):
    with env(**({"HEC_TILE_SKIP": 1} if force else {})):
        Ms = hec.from_csr(A)
    with env(HEC_TILE_SKIP=0):
        Mp = hec.from_csr(A)
    assert Ms.info.ell_tile_w == 1 and Mp.info.ell_tile_w == 0
    return Ms, Mp


@pytest.mark.parametrize("n", [1 << 16, (1 << 17) + 333])
def test_tileskip_degree_sorted_default_bitwise(n):
    A = hecgen.degree_sorted(hecgen.powerlaw(n, seed=41))
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    Ms, Mp = pair(A)
    assert Ms.info.ell_tile_skip > 0.05 and Ms.info.ell_grouped == 0  # already in length order
    ys = run(Ms, x)
    assert ys.tobytes() == run(Mp, x).tobytes()
    assert np.all(np.abs(ys - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


def test_tileskip_integer_bitwise_vs_oracle():
    A = hecgen.degree_sorted(hecgen.powerlaw(1 << 17, integer_values=True, seed=42))
    xi = hecgen.vector(A.n_cols, "int", seed=2)
    Ms, _ = pair(A)
    assert run(Ms, xi).tobytes() == oracle.csr_spmv(A, xi).tobytes()


def test_grouping_natural_powerlaw_bitwise():
    # natural order: rows of every length side by side, so the ELL rows are
    # grouped by length inside 1024-row windows first (y written through the
    # permutation) -- bitwise equal to the ungrouped, unskipped product
    A = hecgen.powerlaw((1 << 17) + 4321, seed=43)
    x = hecgen.vector(A.n_cols, "uniform", seed=3)
    assert hec.from_csr(A).info.ell_grouped == 0   # by default only from 2^20 rows on
    with env(HEC_ELL_GROUP=1):
        Mg = hec.from_csr(A)
    assert Mg.info.ell_grouped == 1 and Mg.info.ell_tile_w == 1 and Mg.info.ell_tile_skip > 0.15
    with env(HEC_ELL_GROUP=0, HEC_TILE_SKIP=0):
        Mp = hec.from_csr(A)
    assert Mp.info.ell_grouped == 0 and Mp.info.ell_tile_w == 0
    yg = run(Mg, x)
    assert yg.tobytes() == run(Mp, x).tobytes()
    assert np.all(np.abs(yg - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))
    # hec_export gives back the row-order HEC of the host converter
    e, r = Mg.export(), hec.from_csr(A, device=-1).export()
    for f in ("ell_col", "ell_val", "tail_rows", "tail_ptr", "tail_col", "tail_val"):
        assert getattr(e, f).tobytes() == getattr(r, f).tobytes()


def test_grouping_integer_bitwise_vs_oracle():
    A = hecgen.powerlaw(1 << 17, integer_values=True, seed=47)
    xi = hecgen.vector(A.n_cols, "int", seed=4)
    with env(HEC_ELL_GROUP=1):
        M = hec.from_csr(A)
    assert M.info.ell_grouped == 1
    assert run(M, xi).tobytes() == oracle.csr_spmv(A, xi).tobytes()


def test_grouping_epilogues_and_host_chunks_bitwise():
    # Eq. (2), the diagonal and the Jacobi sweep through the permutation; and
    # hec_spmv_host's chunks (aligned to the grouping windows)
    A = hecgen.powerlaw(3 << 20, seed=48)
    n = A.n_rows
    x = hecgen.vector(n, "uniform", seed=5)
    y0 = hecgen.vector(n, "uniform", seed=6)
    Mg = hec.from_csr(A)
    with env(HEC_ELL_GROUP=0, HEC_TILE_SKIP=0):
        Mp = hec.from_csr(A)
    assert Mg.info.ell_grouped == 1
    outs = []
    for M in (Mg, Mp):
        y = dev(y0)
        M.spmv_axpby(-0.75, dev(x), 0.5, y)
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        M.diag(d)
        xo = torch.empty(n, dtype=torch.float64, device="cuda")
        M.jacobi(d, dev(y0), dev(x), xo, 0.8)
        torch.cuda.synchronize()
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.full((n,), float("nan"), dtype=torch.float64).pin_memory()
        M.spmv_host(xh, yh)
        outs.append((y.cpu().numpy().tobytes(), d.cpu().numpy().tobytes(), xo.cpu().numpy().tobytes(),
                     yh.numpy().tobytes()))
    assert outs[0] == outs[1]


def test_tileskip_epilogues_bitwise():
    A = hecgen.degree_sorted(hecgen.powerlaw(1 << 16, seed=44))
    n = A.n_rows
    x = hecgen.vector(n, "uniform", seed=5)
    y0 = hecgen.vector(n, "uniform", seed=6)
    Ms, Mp = pair(A)
    outs = []
    for M in (Ms, Mp):
        y = dev(y0)
        M.spmv_axpby(-0.75, dev(x), 0.5, y)  # Eq. (2)
        d = torch.empty(n, dtype=torch.float64, device="cuda")
        M.diag(d)
        xo = torch.empty(n, dtype=torch.float64, device="cuda")
        M.jacobi(d, dev(y0), dev(x), xo, 0.8)  # damped Jacobi (A22)
        torch.cuda.synchronize()
        outs.append((y.cpu().numpy().tobytes(), xo.cpu().numpy().tobytes()))
    assert outs[0] == outs[1]


def test_tileskip_host_chunks_bitwise():
    # >= 2M rows: hec_spmv_host's row chunks start at row offsets (multiples of 512)
    A = hecgen.degree_sorted(hecgen.powerlaw(3 << 20, seed=45))
    x = hecgen.vector(A.n_cols, "uniform", seed=7)
    Ms, Mp = pair(A)
    yp = run(Mp, x)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.full((A.n_rows,), float("nan"), dtype=torch.float64).pin_memory()
    Ms.spmv_host(xh, yh)
    assert yh.numpy().tobytes() == yp.tobytes()


@pytest.mark.parametrize("P", [2, 4])
def test_tileskip_distributed_bitwise(P):
    A = hecgen.degree_sorted(hecgen.powerlaw(1 << 16, seed=46))
    x = hecgen.vector(A.n_cols, "uniform", seed=8)
    plan = hec.partition(A, P, hec.PART_CONTIG_NNZ)
    pp = plan.part_ptr()
    ys = {}
    for flag in (1, 0):
        with env(HEC_TILE_SKIP=flag):
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


def test_grouping_full_size_powerlaw_every_row():
    # configs[4] (2^23 rows): grouped by default, every row bitwise equal to
    # the ungrouped product and within tolerance of the oracle
    A = hecgen.powerlaw(1 << 23, seed=1)
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    Mg = hec.from_csr(A)
    assert Mg.info.ell_grouped == 1 and Mg.info.ell_tile_w == 1
    yg = run(Mg, x)
    Mg.free()
    with env(HEC_ELL_GROUP=0, HEC_TILE_SKIP=0):
        Mp = hec.from_csr(A)
    assert yg.tobytes() == run(Mp, x).tobytes()
    assert np.all(np.abs(yg - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))


@pytest.mark.parametrize("P", [2, 3])
def test_grouping_distributed_submatrices_bitwise(P):
    # sub-matrices of >= 2^16 rows are grouped too: the ELL launch writes each
    # stored row's own output row (row map / offset composed with the grouping)
    A = hecgen.powerlaw(1 << 18, seed=49)
    x = hecgen.vector(A.n_cols, "uniform", seed=9)
    plan = hec.partition(A, P, hec.PART_CONTIG_NNZ)
    pp = plan.part_ptr()
    ys = {}
    for flag in (1, 0):
        with env(HEC_ELL_GROUP=flag, HEC_TILE_SKIP=flag):
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
