"""Input generators (hecgen): the degree-sorted stress variant (SURVEY §8(d)
power-law recipe) is the symmetric permutation P A P^T with rows in
descending length order -- checked against scipy's own row/column indexing."""
import numpy as np
import pytest
import scipy.sparse as sp

import hecgen
import oracle


def _sp(A):
    return sp.csr_matrix((A.val, A.col, A.row_ptr), shape=(A.n_rows, A.n_cols))


@pytest.mark.parametrize("maker", [lambda: hecgen.powerlaw(5000, seed=4),
                                   lambda: hecgen.powerlaw(3000, integer_values=True, seed=7),
                                   lambda: hecgen.spe10(10, 12, 6, seed=3)])
def test_degree_sorted_is_symmetric_permutation(maker):
    A = maker()
    B = hecgen.degree_sorted(A)
    p = B.perm
    assert np.array_equal(np.sort(p), np.arange(A.n_rows))
    L = np.diff(B.row_ptr)
    assert np.all(np.diff(L) <= 0)                       # descending lengths
    La = np.diff(A.row_ptr)
    ties = L[:-1] == L[1:]
    assert np.all(p[:-1][ties] < p[1:][ties])            # stable
    assert np.array_equal(L, La[p])
    assert (abs(_sp(A)[p][:, p] - _sp(B))).max() == 0.0  # B = P A P^T exactly
    assert oracle.is_canonical(B)                        # sorted, unique columns per row
    # diagonal stays on the diagonal
    d = _sp(A).diagonal()
    assert np.array_equal(_sp(B).diagonal(), d[p])


def test_degree_sorted_spmv_commutes_with_permutation():
    A = hecgen.powerlaw(4000, integer_values=True, seed=11)
    B = hecgen.degree_sorted(A)
    x = hecgen.vector(A.n_cols, "int", seed=3)
    # (P A P^T)(P x) = P (A x), exactly in the integer regime (P3)
    assert np.array_equal(oracle.csr_spmv(B, x[B.perm]), oracle.csr_spmv(A, x)[B.perm])


def test_degree_sorted_rejects_rectangular():
    A = hecgen.random_csr(5, 7, 0.5, seed=1)
    with pytest.raises(ValueError):
        hecgen.degree_sorted(A)
