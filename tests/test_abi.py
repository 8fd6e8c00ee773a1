"""The C ABI (include/hec.h) on a CPU-only box: the library loads, exports every
declared symbol, validates inputs with the documented status codes, and refuses
compute on host-only handles (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import hecgen
import paper_1606_00545_b200 as hec
from paper_1606_00545_b200 import hec as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "hec.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hec_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = hec.load()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), f"libhec.so does not export {n}"
    assert set(names) == set(hec.EXPORTED)
    assert b"sm_100a" in L.hec_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", hec.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_opts_default_matches_paper():
    o = H.OptsT()
    hec.load().hec_opts_default(ctypes.byref(o))
    assert (o.width_policy, o.cap, o.stride_unit) == (hec.WIDTH_BG3, 20, 256)


@pytest.mark.parametrize("rows,status", [
    ([[(2, 1.0), (0, 1.0)]], 2),          # unsorted columns
    ([[(1, 1.0), (1, 2.0)]], 2),          # duplicate column
    ([[(3, 1.0)]], 2),                    # column out of range
    ([[(-1, 1.0)]], 2),                   # negative column
])
def test_from_csr_rejects_noncanonical(rows, status):
    A = hecgen.from_rows(3, rows)
    with pytest.raises(hec.HecError) as e:
        hec.from_csr(A, device=-1)
    assert e.value.status == status


def test_from_csr_rejects_bad_row_ptr():
    A = hecgen.from_dense(np.eye(3))
    A.row_ptr = np.array([0, 2, 1, 3], np.int32)
    with pytest.raises(hec.HecError) as e:
        hec.from_csr(A, device=-1)
    assert e.value.status == 2
    A.row_ptr = np.array([1, 1, 2, 3], np.int32)
    with pytest.raises(hec.HecError) as e:
        hec.from_csr(A, device=-1)
    assert e.value.status == 2


def test_bad_options():
    A = hecgen.poisson2d(4, 4)
    for o in (hec.opts(stride_unit=48), hec.opts(stride_unit=0), hec.opts(width_policy=7), hec.opts(cap=-1)):
        with pytest.raises(hec.HecError) as e:
            hec.from_csr(A, o, device=-1)
        assert e.value.status == 1


def test_host_only_handle_refuses_compute():
    A = hecgen.poisson2d(4, 4)
    M = hec.from_csr(A, device=-1)
    assert M.info.device == -1
    L = hec.load()
    x = np.ones(16)
    y = np.empty(16)
    st = L.hec_spmv(M.handle, x.ctypes.data, y.ctypes.data, None)
    assert st == 9                                                 # HEC_ERR_NODEV
    assert b"no CPU fallback" in L.hec_last_error()
    assert L.hec_spmv_host(M.handle, x.ctypes.data, y.ctypes.data, None) == 9


def test_partition_errors():
    A = hecgen.poisson3d(4, 4, 4)
    with pytest.raises(hec.HecError) as e:
        hec.partition(A, 0)
    assert e.value.status == 4
    with pytest.raises(hec.HecError) as e:
        hec.partition(A, 65)
    assert e.value.status == 4
    with pytest.raises(hec.HecError) as e:
        hec.partition(A, 5, hec.PART_GRID, (4, 4, 4))     # more parts than planes
    assert e.value.status == 4
    with pytest.raises(hec.HecError) as e:
        hec.partition(A, 2, hec.PART_GRID, (4, 4, 3))     # grid does not match n
    assert e.value.status == 4
    R = hecgen.random_csr(5, 7, 0.5, seed=1)
    with pytest.raises(hec.HecError) as e:
        hec.partition(R, 2)                                 # distributed mode needs square A (A14)
    assert e.value.status == 3


def test_plan_part_hec_rejects_other_matrix():
    A = hecgen.poisson3d(4, 4, 4)
    P = hec.partition(A, 2, hec.PART_GRID, (4, 4, 4))
    B = hecgen.poisson3d(4, 4, 3)
    with pytest.raises(hec.HecError) as e:
        P.part_hec(B, 0, hec.SUB_ALL)
    assert e.value.status == 8


def test_dist_create_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    A = hecgen.poisson3d(4, 4, 4)
    P = hec.partition(A, 1)
    with pytest.raises(hec.HecError) as e:
        hec.Dist(A, P, 0, None, 0)
    assert e.value.status in (5, 9)


def test_matrix_info_layout_of_the_round2_fields():
    # hec_matrix_info grew fields in round 2 (x-ring, index compression, slot
    # skipping, row grouping): on a host-only handle they read as "off", and
    # the struct the binding declares is exactly as large as the C one (the
    # last field lands where C puts it, or the values below would be garbage)
    import ctypes
    A = hecgen.powerlaw(3000, seed=12)
    inf = hec.from_csr(A, device=-1).info
    assert inf.n_rows == 3000 and inf.device == -1
    assert inf.tail_ring == 0 and inf.ell_idx16 == 0 and inf.ell_tile_w == 0 and inf.ell_grouped == 0
    assert inf.tail_ring_cover == 0.0 and inf.ell_idx16_escaped == -1.0 and inf.ell_tile_skip == 0.0
    assert ctypes.sizeof(type(inf)) % 8 == 0
