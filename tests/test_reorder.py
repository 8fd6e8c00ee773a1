"""NEXT-4 reordering (reading A21): the oracle RCM / permutation
(oracle/reorder_ref.py) pinned to bandwidth closed forms, scipy's
reverse_cuthill_mckee and the permutation identity; the product
(hec_reorder_rcm / hec_permute) bit-exact against the oracle.  CPU only."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

import hecgen
import oracle
import paper_1606_00545_b200 as hec
from oracle import reorder_ref as R


def scramble(A, seed):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(A.n_rows).astype(np.int32)
    return R.permute(A, perm, hecgen.Csr), perm


def tridiag(n):
    rows = []
    for i in range(n):
        r = [(i - 1, -1.0)] if i > 0 else []
        r.append((i, 2.0))
        if i < n - 1:
            r.append((i + 1, -1.0))
        rows.append(r)
    return hecgen.from_rows(n, rows)


def test_path_graph_recovers_bandwidth_one():
    # closed form: a scrambled path graph has an ordering of bandwidth 1, and
    # Cuthill-McKee from a peripheral vertex finds it
    S, _ = scramble(tridiag(200), 1)
    assert R.bandwidth(S) > 10
    p = R.rcm(S)
    assert sorted(p.tolist()) == list(range(200))
    assert R.bandwidth(R.permute(S, p, hecgen.Csr)) == 1


@pytest.mark.parametrize("maker", [lambda: hecgen.poisson2d(20, 15), lambda: hecgen.poisson3d(8, 7, 6),
                                   lambda: hecgen.powerlaw(2000, lmin=3, lmax=8, alpha=2.0, band=6, p_local=1.0, seed=2)])
def test_bandwidth_comparable_to_scipy(maker):
    S, _ = scramble(maker(), 3)
    ours = R.bandwidth(R.permute(S, R.rcm(S), hecgen.Csr))
    M = sp.csr_matrix((S.val, S.col, S.row_ptr), shape=(S.n_rows, S.n_cols))
    q = reverse_cuthill_mckee(M, symmetric_mode=False)
    theirs = R.bandwidth(R.permute(S, q.astype(np.int32), hecgen.Csr))
    assert ours <= 1.5 * theirs + 2
    assert ours < R.bandwidth(S) / 2


def test_disconnected_components_and_permutation_identity():
    D = np.zeros((9, 9))
    D[:4, :4] = np.diag([2.0] * 4) + np.diag([1.0] * 3, 1) + np.diag([1.0] * 3, -1)
    D[4:, 4:] = 3.0 * np.eye(5) + np.diag([1.0] * 4, 1) + np.diag([1.0] * 4, -1)
    A, _ = scramble(hecgen.from_dense(D), 5)
    p = R.rcm(A)
    assert sorted(p.tolist()) == list(range(9))
    B = R.permute(A, p, hecgen.Csr)
    x = np.arange(9, dtype=np.float64) - 4
    # (P A P^T)(P x) = P (A x), exactly on integer data
    assert oracle.csr_spmv(B, x[p]).tolist() == oracle.csr_spmv(A, x)[p].tolist()
    assert R.bandwidth(B) == 1


@pytest.mark.parametrize("maker", [lambda: hecgen.random_csr(60, 60, 0.05, seed=3),
                                   lambda: hecgen.powerlaw(1500, seed=4),
                                   lambda: hecgen.spe10(10, 12, 6, seed=2),
                                   lambda: scramble(hecgen.poisson3d(9, 8, 7), 9)[0]])
def test_product_matches_oracle_bitexact(maker):
    A = maker()
    p = hec.reorder_rcm(A)
    assert p.tolist() == R.rcm(A).tolist()
    B = hec.permute(A, p)
    Bo = R.permute(A, p, hecgen.Csr)
    for f in ("row_ptr", "col", "val"):
        assert getattr(B, f).tobytes() == getattr(Bo, f).tobytes()


def test_rcm_shrinks_scrambled_halo():
    # the point of P:149: after reordering, contiguous partitions exchange far less
    S, _ = scramble(hecgen.poisson3d(12, 12, 12), 7)
    B = hec.permute(S, hec.reorder_rcm(S))
    halo = lambda M: sum(len(hec.partition(M, 4, hec.PART_CONTIG_ROWS).export(p).recv_cols) for p in range(4))  # noqa: E731
    assert halo(B) * 5 < halo(S)


def test_errors():
    R5 = hecgen.random_csr(5, 7, 0.5, seed=1)
    with pytest.raises(hec.HecError) as e:
        hec.reorder_rcm(R5)
    assert e.value.status == 3
    A = hecgen.poisson2d(3, 3)
    with pytest.raises(hec.HecError) as e:
        hec.permute(A, np.zeros(9, np.int32))
    assert e.value.status == 1
