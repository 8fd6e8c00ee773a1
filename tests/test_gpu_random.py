"""Randomised GPU parity sweep: many small seeded matrices -- random shapes
(square and rectangular), densities, row-length mixes (power-law, empty rows,
single long rows), width policies (BG3 / CAP / FIXED), stride units and tail
schedules (entries per lane, small tails first or last) -- each compared with
the serial C oracle on every row (north_star tolerance; bitwise on integer
data), and hec_export compared with the host-only handle (the HEC arrays
bit-exact against the host converter).  Complements the structured cases of
test_gpu_spmv.py / test_gpu_tail.py with combinations nobody picked by hand."""
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


def random_case(seed):
    rng = np.random.default_rng(seed)
    kind = seed % 4
    if kind == 0:
        n = int(rng.integers(1, 3000))
        A = hecgen.random_csr(n, int(rng.integers(1, 3000)), float(rng.uniform(0.0005, 0.02)),
                              integer_values=bool(rng.integers(0, 2)), seed=seed)
    elif kind == 1:
        A = hecgen.powerlaw(int(rng.integers(200, 20000)), integer_values=bool(rng.integers(0, 2)), seed=seed)
    elif kind == 2:  # explicit rows: empties, one very long row, short rows
        n_cols = int(rng.integers(50, 5000))
        rows = []
        for i in range(int(rng.integers(1, 400))):
            r = rng.random()
            L = 0 if r < 0.2 else (int(rng.integers(1, n_cols + 1)) if r > 0.97 else int(rng.integers(1, 12)))
            cols = np.sort(rng.choice(n_cols, size=min(L, n_cols), replace=False))
            rows.append([(int(c), float(rng.integers(-8, 9)) or 1.0) for c in cols])
        A = hecgen.from_rows(n_cols, rows)
    else:
        A = hecgen.spe10(int(rng.integers(3, 20)), int(rng.integers(3, 20)), int(rng.integers(2, 8)), seed=seed)
    policy = int(rng.integers(0, 3))
    unit = int(rng.choice([32, 64, 256, 512]))
    o = hec.opts(policy, int(rng.integers(0, 25)), int(rng.integers(0, 12)), unit)
    env = {"HEC_TAIL_EPL": str(int(rng.choice([1, 2, 4, 8, 16, 32, 64]))),
           "HEC_FUSE_TAIL": str(int(rng.integers(0, 2)))}
    return A, o, env


@pytest.mark.parametrize("seed", range(48))
def test_random_matrix_parity(seed):
    A, o, env = random_case(seed)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        M = hec.from_csr(A, o)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    integer = np.all(A.val == np.round(A.val)) if A.nnz else True
    x = hecgen.vector(A.n_cols, "int" if integer else "uniform", seed=seed)
    xd = torch.from_numpy(x).cuda()
    yd = torch.full((A.n_rows,), float("nan"), dtype=torch.float64, device="cuda")
    M.spmv(xd, yd)
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    ref = oracle.csr_spmv(A, x)
    if integer:
        assert y.tobytes() == ref.tobytes(), (seed, env)
    else:
        assert np.all(np.abs(y - ref) <= oracle.tolerance(A, x)), (seed, env)
    e, r = M.export(), hec.from_csr(A, o, device=-1).export()
    for f in ("ell_col", "ell_val", "tail_rows", "tail_ptr", "tail_col", "tail_val"):
        assert getattr(e, f).tobytes() == getattr(r, f).tobytes(), (seed, f)
