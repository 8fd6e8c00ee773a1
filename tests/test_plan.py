"""Partition + halo plan (libhec host planner) vs the oracle O3, BIT-EXACT
(BASELINE.json north_star: "the halo index lists must match bit-exactly"),
and each part's interior/boundary sub-HECs vs O2 applied to the oracle's local
matrices with the partition width (reading A12)."""
import numpy as np
import pytest

import hecgen
import paper_1606_00545_b200 as hec
from oracle import hec_ref as H
from oracle import plan_ref as PR


def check_plan(A, P, kind, grid=None, opts_args=(0, 20, 0, 256), check_sub=True):
    ref_pp = PR.part_ptr_ref(A, P, kind, grid)
    plan = hec.partition(A, P, kind, grid)
    assert plan.part_ptr().tolist() == ref_pp.tolist()
    parts = PR.plan_ref(A, ref_pp)
    o = hec.opts(*opts_args)
    for p, ref in enumerate(parts):
        got = plan.export(p, o)
        assert (got.r0, got.r1) == (ref.r0, ref.r1)
        for f, g in (("recv_cols", "recv"), ("recv_off", "recv_off"), ("send_idx", "send_idx"),
                     ("send_off", "send_off"), ("interior", "interior"), ("boundary", "boundary")):
            assert getattr(got, f).tolist() == getattr(ref, g).tolist(), (p, f)
        w = PR.part_width(ref, hecgen.Csr, opts_args[0], opts_args[1], opts_args[2])
        assert got.width == w
        if not check_sub:
            continue
        for which, name in ((hec.SUB_INTERIOR, "interior"), (hec.SUB_BOUNDARY, "boundary"), (hec.SUB_ALL, "all")):
            L = PR.local_csr(ref, name, hecgen.Csr)
            r = H.build(L, stride_unit=opts_args[3], width=w)
            M = plan.part_hec(A, p, which, o, device=-1)
            e = M.export()
            assert (e.width, e.stride) == (r.width, r.stride)
            for f in ("ell_col", "ell_val", "tail_rows", "tail_ptr", "tail_col", "tail_val"):
                assert getattr(e, f).tobytes() == getattr(r, f).tobytes(), (p, name, f)
    return plan, parts


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_poisson_grid_slabs(P):
    check_plan(hecgen.poisson3d(8, 6, 8), P, hec.PART_GRID, (8, 6, 8))


@pytest.mark.parametrize("P", [1, 2, 5])
def test_poisson2d_grid(P):
    check_plan(hecgen.poisson2d(9, 7), P, hec.PART_GRID, (9, 7, 1))


@pytest.mark.parametrize("P,kind", [(2, hec.PART_CONTIG_NNZ), (3, hec.PART_CONTIG_NNZ), (8, hec.PART_CONTIG_NNZ),
                                    (4, hec.PART_CONTIG_ROWS), (16, hec.PART_CONTIG_ROWS)])
def test_powerlaw_parts(P, kind):
    check_plan(hecgen.powerlaw(600, seed=P), P, kind)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_contig_cost_parts(P):
    check_plan(hecgen.powerlaw(600, seed=P), P, hec.PART_CONTIG_COST)


@pytest.mark.parametrize("P", [4, 8])
def test_contig_cost_degree_sorted(P):
    check_plan(hecgen.degree_sorted(hecgen.powerlaw(2000, seed=5)), P, hec.PART_CONTIG_COST, check_sub=False)


def test_contig_cost_p_equals_n():
    check_plan(hecgen.random_csr(12, 12, 0.3, seed=4), 12, hec.PART_CONTIG_COST)


def test_policies_and_units():
    A = hecgen.powerlaw(300, seed=4)
    for args in [(1, 20, 0, 32), (0, 5, 0, 256), (2, 0, 3, 64), (1, 0, 0, 256)]:
        check_plan(A, 3, hec.PART_CONTIG_NNZ, opts_args=args)


def test_random_and_degenerate():
    check_plan(hecgen.random_csr(40, 40, 0.1, seed=3), 7, hec.PART_CONTIG_NNZ)
    check_plan(hecgen.random_csr(12, 12, 0.3, seed=4), 12, hec.PART_CONTIG_ROWS)   # P = n
    D = np.zeros((12, 12))
    for b in range(3):
        D[4 * b:4 * b + 4, 4 * b:4 * b + 4] = 1.0
    plan, _ = check_plan(hecgen.from_dense(D), 3, hec.PART_CONTIG_ROWS)          # no halo
    for p in range(3):
        inf = plan.part_info(p)
        assert inf.n_halo == 0 and inf.n_boundary == 0 and inf.n_send == 0


def test_spe10_parts():
    check_plan(hecgen.spe10(12, 20, 9, seed=4), 4, hec.PART_CONTIG_NNZ)


def test_256_slab_closed_forms_from_product():
    # 256^3 z-slabs at P = 8 (closed forms): recv = 65,536 per
    # neighbour; boundary = first/last plane.  Only the product plan runs at
    # this size (the oracle's Python loops are for small inputs).
    A = hecgen.poisson3d(256, 256, 256)
    plan = hec.partition(A, 8, hec.PART_GRID, (256, 256, 256))
    plane = 256 * 256
    for p in range(8):
        a = plan.export(p)
        nb = [q for q in (p - 1, p + 1) if 0 <= q < 8]
        assert len(a.recv_cols) == plane * len(nb)
        assert a.r1 - a.r0 == 32 * plane
        exp_b = (list(range(plane)) if p > 0 else []) + (list(range(31 * plane, 32 * plane)) if p < 7 else [])
        assert a.boundary.tolist() == exp_b
        assert a.width == 7
        if p > 0:
            assert a.recv_cols[:plane].tolist() == list(range(a.r0 - plane, a.r0))
        if p < 7:
            assert a.recv_cols[-plane:].tolist() == list(range(a.r1, a.r1 + plane))
            assert a.send_idx[a.send_off[p + 1]:a.send_off[p + 2]].tolist() == list(range(31 * plane, 32 * plane))
