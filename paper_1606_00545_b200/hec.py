"""Thin ctypes binding of libhec.so (include/hec.h) -- argument marshalling only.

Every step of the SpMV path runs inside libhec.so (host converter/planner in
C++, kernels in CUDA for sm_100a).  PyTorch supplies device memory, streams and
process groups.  There is no CPU fallback: if the library cannot be loaded the
import fails, and compute on a host-only handle raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _build

# ----------------------------------------------------------------- loading --
_lib = None


class HecError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hec status {status}: {msg}")
        self.status = status


STATUS = {0: "HEC_OK", 1: "HEC_ERR_ARG", 2: "HEC_ERR_FORMAT", 3: "HEC_ERR_DIM", 4: "HEC_ERR_PARTS",
          5: "HEC_ERR_CUDA", 6: "HEC_ERR_NCCL", 7: "HEC_ERR_NOMEM", 8: "HEC_ERR_STATE", 9: "HEC_ERR_NODEV"}
WIDTH_BG3, WIDTH_CAP, WIDTH_FIXED = 0, 1, 2
PART_CONTIG_NNZ, PART_CONTIG_ROWS, PART_GRID, PART_CONTIG_COST, PART_EXPLICIT = 0, 1, 2, 3, 4
ORDER_BISECT, ORDER_MULTILEVEL = 0, 1
SUB_INTERIOR, SUB_BOUNDARY, SUB_ALL = 0, 1, 2
NCCL_ID_BYTES = 128
IPC_BYTES = 64

i32, i64, vp, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double


class CsrT(ctypes.Structure):
    _fields_ = [("n_rows", i32), ("n_cols", i32), ("nnz", i64),
                ("row_ptr", vp), ("col_idx", vp), ("val", vp)]


class OptsT(ctypes.Structure):
    _fields_ = [("width_policy", i32), ("cap", i32), ("fixed_width", i32), ("stride_unit", i32)]


class MatrixInfoT(ctypes.Structure):
    _fields_ = [("n_rows", i32), ("n_cols", i32), ("ell_width", i32), ("ell_stride", i32),
                ("nnz", i64), ("ell_nnz", i64), ("tail_rows", i32), ("tail_group", i32),
                ("tail_nnz", i64), ("device_bytes", i64), ("device", i32), ("tail_fused", i32),
                ("tail_ring", i32), ("ell_idx16", i32), ("tail_ring_cover", ctypes.c_double),
                ("ell_idx16_escaped", ctypes.c_double), ("ell_tile_skip", ctypes.c_double),
                ("ell_tile_w", i32), ("ell_grouped", i32)]


class HostArraysT(ctypes.Structure):
    _fields_ = [("ell_col", vp), ("ell_val", vp), ("tail_rows", vp), ("tail_ptr", vp),
                ("tail_col", vp), ("tail_val", vp)]


class PartInfoT(ctypes.Structure):
    _fields_ = [("r0", i32), ("r1", i32), ("n_halo", i32), ("n_send", i32), ("n_interior", i32),
                ("n_boundary", i32), ("n_recv_peers", i32), ("n_send_peers", i32), ("width", i32),
                ("reserved", i32)]


class PlanArraysT(ctypes.Structure):
    _fields_ = [("recv_cols", vp), ("recv_off", vp), ("send_idx", vp), ("send_off", vp),
                ("interior", vp), ("boundary", vp)]


class DistInfoT(ctypes.Structure):
    _fields_ = [("rank", i32), ("n_parts", i32), ("r0", i32), ("r1", i32), ("n_halo", i32),
                ("n_send", i32), ("n_interior", i32), ("n_boundary", i32), ("width", i32),
                ("launches", i32), ("device_bytes", i64), ("algorithmic_bytes", i64),
                ("nnz_local", i64)]


EXPORTED = [
    "hec_last_error", "hec_version", "hec_opts_default", "hec_from_csr", "hec_info", "hec_export",
    "hec_spmv", "hec_spmv_host", "hec_spmv_launches", "hec_free", "hec_partition",
    "hec_plan_n_parts", "hec_plan_part_ptr", "hec_plan_part_info", "hec_plan_part_info_opts",
    "hec_plan_export", "hec_plan_part_hec", "hec_plan_free", "hec_nccl_unique_id",
    "hec_dist_create", "hec_dist_create_local", "hec_spmv_dist", "hec_spmv_dist_local",
    "hec_dist_get_info", "hec_dist_free", "hec_dist_create_p2p", "hec_dist_p2p_connect",
    "hec_dist_enable_p2p", "hec_dist_p2p_connect_local", "hec_dist_check",
    "hec_spmv_axpby", "hec_diag", "hec_jacobi", "hec_axpby", "hec_axpbyz", "hec_dot", "hec_norm2", "hec_bicgstab", "hec_cg",
    "hec_bicgstab_dist", "hec_cg_dist", "hec_from_csr_hyb", "hec_reorder_rcm", "hec_permute",
    "hec_spmv_dist_host", "hec_dist_comm_size", "hec_bicgstab_dist_local", "hec_cg_dist_local",
    "hec_partition_order", "hec_dist_set_timing", "hec_dist_phase_times",
]


class SolveInfoT(ctypes.Structure):
    _fields_ = [("iterations", i32), ("converged", i32), ("breakdown", i32), ("reserved", i32),
                ("rel_residual", dbl)]


def lib_path() -> str:
    return _build.LIB


def load(build: bool = True):
    """Load libhec.so (building it in-tree first if stale).  Import torch
    before calling this so the process shares torch's libnccl.so.2."""
    global _lib
    if _lib is not None:
        return _lib
    try:
        import torch  # noqa: F401  (maps torch's NCCL/cudart first)
    except Exception:
        pass
    path = _build.build() if build else _build.LIB
    if not os.path.exists(path):
        raise ImportError(f"libhec.so not built at {path}")
    L = ctypes.CDLL(path)
    st = ctypes.c_int
    L.hec_last_error.restype = ctypes.c_char_p
    L.hec_version.restype = ctypes.c_char_p
    L.hec_opts_default.restype = None
    L.hec_opts_default.argtypes = [ctypes.POINTER(OptsT)]
    for f in (L.hec_from_csr, L.hec_from_csr_hyb):
        f.restype = st
        f.argtypes = [ctypes.POINTER(CsrT), ctypes.POINTER(OptsT), i32, vp, ctypes.POINTER(vp)]
    L.hec_info.restype = st
    L.hec_info.argtypes = [vp, ctypes.POINTER(MatrixInfoT)]
    L.hec_export.restype = st
    L.hec_export.argtypes = [vp, ctypes.POINTER(HostArraysT)]
    L.hec_spmv.restype = st
    L.hec_spmv.argtypes = [vp, vp, vp, vp]
    L.hec_spmv_host.restype = st
    L.hec_spmv_host.argtypes = [vp, vp, vp, vp]
    L.hec_spmv_launches.restype = i32
    L.hec_spmv_launches.argtypes = [vp]
    L.hec_free.restype = None
    L.hec_free.argtypes = [vp]
    L.hec_partition.restype = st
    L.hec_partition.argtypes = [ctypes.POINTER(CsrT), i32, i32, vp, ctypes.POINTER(vp)]
    L.hec_plan_n_parts.restype = st
    L.hec_plan_n_parts.argtypes = [vp, ctypes.POINTER(i32)]
    L.hec_plan_part_ptr.restype = st
    L.hec_plan_part_ptr.argtypes = [vp, vp]
    L.hec_plan_part_info.restype = st
    L.hec_plan_part_info.argtypes = [vp, i32, ctypes.POINTER(PartInfoT)]
    L.hec_plan_part_info_opts.restype = st
    L.hec_plan_part_info_opts.argtypes = [vp, i32, ctypes.POINTER(OptsT), ctypes.POINTER(PartInfoT)]
    L.hec_plan_export.restype = st
    L.hec_plan_export.argtypes = [vp, i32, ctypes.POINTER(PlanArraysT)]
    L.hec_plan_part_hec.restype = st
    L.hec_plan_part_hec.argtypes = [vp, ctypes.POINTER(CsrT), i32, i32, ctypes.POINTER(OptsT), i32, vp,
                                    ctypes.POINTER(vp)]
    L.hec_plan_free.restype = None
    L.hec_plan_free.argtypes = [vp]
    L.hec_nccl_unique_id.restype = st
    L.hec_nccl_unique_id.argtypes = [vp]
    L.hec_dist_create.restype = st
    L.hec_dist_create.argtypes = [ctypes.POINTER(CsrT), vp, ctypes.POINTER(OptsT), i32, vp, i32,
                                  ctypes.POINTER(vp)]
    L.hec_dist_create_local.restype = st
    L.hec_dist_create_local.argtypes = [ctypes.POINTER(CsrT), vp, ctypes.POINTER(OptsT), i32, vp]
    L.hec_spmv_dist.restype = st
    L.hec_spmv_dist.argtypes = [vp, vp, vp, vp]
    L.hec_spmv_dist_host.restype = st
    L.hec_spmv_dist_host.argtypes = [vp, vp, vp, vp]
    L.hec_dist_set_timing.restype = st
    L.hec_dist_set_timing.argtypes = [vp, i32]
    L.hec_dist_phase_times.restype = st
    L.hec_dist_phase_times.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
    L.hec_dist_comm_size.restype = st
    L.hec_dist_comm_size.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.hec_spmv_dist_local.restype = st
    L.hec_spmv_dist_local.argtypes = [vp, i32, vp, vp, vp]
    L.hec_dist_get_info.restype = st
    L.hec_dist_get_info.argtypes = [vp, ctypes.POINTER(DistInfoT)]
    L.hec_dist_free.restype = None
    L.hec_dist_free.argtypes = [vp]
    L.hec_dist_create_p2p.restype = st
    L.hec_dist_create_p2p.argtypes = [ctypes.POINTER(CsrT), vp, ctypes.POINTER(OptsT), i32, i32,
                                      ctypes.POINTER(vp), vp]
    L.hec_dist_p2p_connect.restype = st
    L.hec_dist_p2p_connect.argtypes = [vp, vp]
    L.hec_dist_enable_p2p.restype = st
    L.hec_dist_enable_p2p.argtypes = [vp]
    L.hec_dist_p2p_connect_local.restype = st
    L.hec_dist_p2p_connect_local.argtypes = [vp, i32]
    L.hec_dist_check.restype = st
    L.hec_dist_check.argtypes = [vp]
    L.hec_spmv_axpby.restype = st
    L.hec_spmv_axpby.argtypes = [vp, dbl, vp, dbl, vp, vp]
    L.hec_diag.restype = st
    L.hec_diag.argtypes = [vp, vp, vp]
    L.hec_jacobi.restype = st
    L.hec_jacobi.argtypes = [vp, vp, vp, vp, vp, dbl, vp]
    L.hec_axpby.restype = st
    L.hec_axpby.argtypes = [i64, dbl, vp, dbl, vp, vp]
    L.hec_axpbyz.restype = st
    L.hec_axpbyz.argtypes = [i64, dbl, vp, dbl, vp, vp, vp]
    L.hec_dot.restype = st
    L.hec_dot.argtypes = [i64, vp, vp, ctypes.POINTER(dbl), vp]
    L.hec_norm2.restype = st
    L.hec_norm2.argtypes = [i64, vp, ctypes.POINTER(dbl), vp]
    L.hec_reorder_rcm.restype = st
    L.hec_reorder_rcm.argtypes = [ctypes.POINTER(CsrT), vp]
    L.hec_partition_order.restype = st
    L.hec_partition_order.argtypes = [ctypes.POINTER(CsrT), i32, i32, vp, vp]
    L.hec_permute.restype = st
    L.hec_permute.argtypes = [ctypes.POINTER(CsrT), vp, vp, vp, vp]
    for f in (L.hec_bicgstab, L.hec_cg, L.hec_bicgstab_dist, L.hec_cg_dist):
        f.restype = st
        f.argtypes = [vp, vp, vp, dbl, i32, vp, ctypes.POINTER(SolveInfoT)]
    for f in (L.hec_bicgstab_dist_local, L.hec_cg_dist_local):
        f.restype = st
        f.argtypes = [vp, i32, vp, vp, dbl, i32, vp, ctypes.POINTER(SolveInfoT)]
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        msg = _lib.hec_last_error().decode(errors="replace")
        raise HecError(status, f"{STATUS.get(status, '?')}: {msg}")


def _p(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


# ------------------------------------------------------------------- inputs --
class _CsrArgs:
    """Keeps contiguous int32/float64 copies alive while a call borrows them."""

    def __init__(self, A):
        self.row_ptr = np.ascontiguousarray(A.row_ptr, dtype=np.int32)
        self.col = np.ascontiguousarray(A.col, dtype=np.int32)
        self.val = np.ascontiguousarray(A.val, dtype=np.float64)
        self.s = CsrT(int(A.n_rows), int(A.n_cols), int(self.col.shape[0]),
                      _p(self.row_ptr), _p(self.col), _p(self.val))

    def ref(self):
        return ctypes.byref(self.s)


def opts(width_policy: int = WIDTH_BG3, cap: int = 20, fixed_width: int = 0,
         stride_unit: int = 256) -> OptsT:
    return OptsT(width_policy, cap, fixed_width, stride_unit)


def _stream_ptr(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dptr(t, n: int, name: str) -> int:
    import torch
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float64 or not t.is_contiguous() or t.numel() < n:
        raise ValueError(f"{name} must be contiguous float64 with >= {n} elements")
    return t.data_ptr()


def _hptr(a, n: int, name: str) -> int:
    """Host buffer pointer: a numpy array or a CPU torch tensor, contiguous
    float64 with >= n elements.  Anything else raises (a converted temporary
    would be freed before the C call reads it)."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"] or a.size < n:
            raise ValueError(f"{name} must be a contiguous float64 array with >= {n} elements")
        return _p(a)
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        if a.device.type != "cpu":
            raise TypeError(f"{name} must be a host (CPU) tensor for spmv_host")
        if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() < n:
            raise ValueError(f"{name} must be contiguous float64 with >= {n} elements")
        return a.data_ptr() if a.numel() else 0
    raise TypeError(f"{name} must be a numpy array or a CPU torch tensor")


@dataclass
class HecArrays:
    width: int
    stride: int
    ell_col: np.ndarray
    ell_val: np.ndarray
    tail_rows: np.ndarray
    tail_ptr: np.ndarray
    tail_col: np.ndarray
    tail_val: np.ndarray


# ------------------------------------------------------------------ matrix --
class Matrix:
    """HEC matrix handle (hec_from_csr).  device=-1 builds a host-only handle
    (for conversion checks without a GPU; compute refuses it)."""

    def __init__(self, A=None, options: OptsT | None = None, device: int = 0, stream=None,
                 _handle: int | None = None, hyb: bool = False):
        L = load()
        self._h = vp()
        if _handle is not None:
            self._h = vp(_handle)
        else:
            args = _CsrArgs(A)
            o = options if options is not None else opts()
            s = _stream_ptr(stream) if device >= 0 else 0
            make = L.hec_from_csr_hyb if hyb else L.hec_from_csr
            _check(make(args.ref(), ctypes.byref(o), device, s, ctypes.byref(self._h)))
        self.info = self._info()

    def _info(self) -> MatrixInfoT:
        inf = MatrixInfoT()
        _check(_lib.hec_info(self._h, ctypes.byref(inf)))
        return inf

    @property
    def handle(self) -> int:
        return self._h.value

    @property
    def n_rows(self) -> int:
        return self.info.n_rows

    @property
    def n_cols(self) -> int:
        return self.info.n_cols

    def export(self) -> HecArrays:
        inf = self.info
        slots = inf.ell_width * inf.ell_stride
        a = HecArrays(inf.ell_width, inf.ell_stride, np.empty(slots, np.int32), np.empty(slots, np.float64),
                      np.empty(inf.tail_rows, np.int32), np.empty(inf.tail_rows + 1, np.int32),
                      np.empty(inf.tail_nnz, np.int32), np.empty(inf.tail_nnz, np.float64))
        h = HostArraysT(_p(a.ell_col), _p(a.ell_val), _p(a.tail_rows), _p(a.tail_ptr), _p(a.tail_col),
                        _p(a.tail_val))
        _check(_lib.hec_export(self._h, ctypes.byref(h)))
        return a

    def spmv(self, x, y, stream=None):
        """y = A x on the device (async on `stream`, default torch's current)."""
        _check(_lib.hec_spmv(self._h, _dptr(x, self.n_cols, "x"), _dptr(y, self.n_rows, "y"),
                             _stream_ptr(stream)))
        return y

    def spmv_host(self, x, y=None, stream=None):
        """y = A x with host buffers (numpy arrays or CPU torch tensors, pinned
        for full PCIe rate); synchronous.  Both must be contiguous float64 with
        at least n_cols / n_rows elements (no conversion copies: the C side
        reads and writes the caller's memory directly)."""
        if y is None:
            y = np.empty(self.n_rows, np.float64)
        xp = _hptr(x, self.n_cols, "x")
        yp = _hptr(y, self.n_rows, "y")
        _check(_lib.hec_spmv_host(self._h, xp, yp, _stream_ptr(stream)))
        return y

    def spmv_axpby(self, alpha: float, x, beta: float, y, stream=None):
        """Eq. (2): y = alpha A x + beta y on the device."""
        _check(_lib.hec_spmv_axpby(self._h, float(alpha), _dptr(x, self.n_cols, "x"), float(beta),
                                   _dptr(y, self.n_rows, "y"), _stream_ptr(stream)))
        return y

    def diag(self, d, stream=None):
        """d[i] = A_ii (+0.0 where row i stores no diagonal entry), on the device."""
        _check(_lib.hec_diag(self._h, _dptr(d, self.n_rows, "d"), _stream_ptr(stream)))
        return d

    def jacobi(self, d, b, x, x_out, omega: float, stream=None):
        """One damped-Jacobi sweep x_out = x + omega D^-1 (b - A x) on the device (A22)."""
        n = self.n_rows
        _check(_lib.hec_jacobi(self._h, _dptr(d, n, "d"), _dptr(b, n, "b"), _dptr(x, n, "x"),
                               _dptr(x_out, n, "x_out"), float(omega), _stream_ptr(stream)))
        return x_out

    def bicgstab(self, b, x, tol: float = 1e-8, max_it: int = 1000, stream=None) -> SolveInfoT:
        """Alg. 4 (unpreconditioned) on the device; x holds x0 on entry."""
        inf = SolveInfoT()
        _check(_lib.hec_bicgstab(self._h, _dptr(b, self.n_rows, "b"), _dptr(x, self.n_cols, "x"), float(tol),
                                 int(max_it), _stream_ptr(stream), ctypes.byref(inf)))
        return inf

    def cg(self, b, x, tol: float = 1e-8, max_it: int = 1000, stream=None) -> SolveInfoT:
        """Conjugate gradients (SPD A) on the device; x holds x0 on entry."""
        inf = SolveInfoT()
        _check(_lib.hec_cg(self._h, _dptr(b, self.n_rows, "b"), _dptr(x, self.n_cols, "x"), float(tol),
                           int(max_it), _stream_ptr(stream), ctypes.byref(inf)))
        return inf

    @property
    def launches(self) -> int:
        return int(_lib.hec_spmv_launches(self._h))

    def free(self):
        if self._h and self._h.value:
            _lib.hec_free(self._h)
            self._h = vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def from_csr(A, options: OptsT | None = None, device: int = 0, stream=None) -> Matrix:
    return Matrix(A, options, device, stream)


def from_csr_hyb(A, options: OptsT | None = None, device: int = 0, stream=None) -> Matrix:
    """ELL + COO (Bell-Garland HYB) comparison variant (NEXT-2)."""
    return Matrix(A, options, device, stream, hyb=True)


# -------------------------------------------------------------------- plan --
@dataclass
class PartArrays:
    r0: int
    r1: int
    width: int
    recv_cols: np.ndarray
    recv_off: np.ndarray
    send_idx: np.ndarray
    send_off: np.ndarray
    interior: np.ndarray
    boundary: np.ndarray


class Plan:
    """Row partition + halo plan (hec_partition); host-only."""

    def __init__(self, A, n_parts: int, kind: int = PART_CONTIG_NNZ, grid=None):
        L = load()
        self._h = vp()
        args = _CsrArgs(A)
        g = (ctypes.c_int32 * len(grid))(*[int(v) for v in grid]) if grid is not None else None
        _check(L.hec_partition(args.ref(), n_parts, kind, ctypes.cast(g, vp) if g is not None else None,
                               ctypes.byref(self._h)))
        self.n_parts = n_parts

    @property
    def handle(self) -> int:
        return self._h.value

    def part_ptr(self) -> np.ndarray:
        pp = np.empty(self.n_parts + 1, np.int32)
        _check(_lib.hec_plan_part_ptr(self._h, _p(pp)))
        return pp

    def part_info(self, part: int, options: OptsT | None = None) -> PartInfoT:
        inf = PartInfoT()
        if options is None:
            _check(_lib.hec_plan_part_info(self._h, part, ctypes.byref(inf)))
        else:
            _check(_lib.hec_plan_part_info_opts(self._h, part, ctypes.byref(options), ctypes.byref(inf)))
        return inf

    def export(self, part: int, options: OptsT | None = None) -> PartArrays:
        inf = self.part_info(part, options)
        P = self.n_parts
        a = PartArrays(inf.r0, inf.r1, inf.width, np.empty(inf.n_halo, np.int32), np.empty(P + 1, np.int32),
                       np.empty(inf.n_send, np.int32), np.empty(P + 1, np.int32),
                       np.empty(inf.n_interior, np.int32), np.empty(inf.n_boundary, np.int32))
        h = PlanArraysT(_p(a.recv_cols), _p(a.recv_off), _p(a.send_idx), _p(a.send_off), _p(a.interior),
                        _p(a.boundary))
        _check(_lib.hec_plan_export(self._h, part, ctypes.byref(h)))
        return a

    def part_hec(self, A, part: int, which: int, options: OptsT | None = None, device: int = -1,
                 stream=None) -> Matrix:
        args = _CsrArgs(A)
        o = options if options is not None else opts()
        h = vp()
        s = _stream_ptr(stream) if device >= 0 else 0
        _check(_lib.hec_plan_part_hec(self._h, args.ref(), part, which, ctypes.byref(o), device, s,
                                      ctypes.byref(h)))
        return Matrix(_handle=h.value)

    def free(self):
        if self._h and self._h.value:
            _lib.hec_plan_free(self._h)
            self._h = vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def partition(A, n_parts: int, kind: int = PART_CONTIG_NNZ, grid=None) -> Plan:
    return Plan(A, n_parts, kind, grid)


# ------------------------------------------------------------- distributed --
def nccl_unique_id() -> bytes:
    load()
    buf = (ctypes.c_uint8 * NCCL_ID_BYTES)()
    _check(_lib.hec_nccl_unique_id(ctypes.cast(buf, vp)))
    return bytes(buf)


class Dist:
    """One rank of the row-partitioned SpMV (hec_dist_create / hec_spmv_dist)."""

    def __init__(self, A=None, plan: Plan | None = None, rank: int = 0, nccl_id: bytes | None = None,
                 device: int = 0, options: OptsT | None = None, _handle: int | None = None):
        load()
        self._h = vp()
        if _handle is not None:
            self._h = vp(_handle)
        else:
            args = _CsrArgs(A)
            o = options if options is not None else opts()
            idbuf = (ctypes.c_uint8 * NCCL_ID_BYTES).from_buffer_copy(nccl_id) if nccl_id else None
            _check(_lib.hec_dist_create(args.ref(), plan.handle, ctypes.byref(o), rank,
                                        ctypes.cast(idbuf, vp) if idbuf is not None else None, device,
                                        ctypes.byref(self._h)))
        self.info = DistInfoT()
        _check(_lib.hec_dist_get_info(self._h, ctypes.byref(self.info)))

    @classmethod
    def create_p2p(cls, A, plan: "Plan", rank: int, device: int = 0,
                   options: OptsT | None = None) -> tuple["Dist", bytes]:
        """No-NCCL rank for the peer-memory transport (hec_dist_create_p2p):
        returns the handle and this rank's window IPC handle; all-gather the
        handles (e.g. torch.distributed) and call p2p_connect."""
        load()
        args = _CsrArgs(A)
        o = options if options is not None else opts()
        h = vp()
        buf = (ctypes.c_uint8 * IPC_BYTES)()
        _check(_lib.hec_dist_create_p2p(args.ref(), plan.handle, ctypes.byref(o), rank, device,
                                        ctypes.byref(h), ctypes.cast(buf, vp)))
        return cls(_handle=h.value), bytes(buf)

    def p2p_connect(self, handles: list[bytes]):
        """Map the neighbours' windows (handles in rank order) and use the peer-memory transport."""
        blob = b"".join(handles)
        if len(blob) != IPC_BYTES * len(handles):
            raise ValueError("each handle must be IPC_BYTES long")
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(_lib.hec_dist_p2p_connect(self._h, ctypes.cast(buf, vp)))
        _check(_lib.hec_dist_get_info(self._h, ctypes.byref(self.info)))

    def enable_p2p(self):
        """COLLECTIVE: switch an NCCL handle's halo exchange to the peer-memory transport."""
        _check(_lib.hec_dist_enable_p2p(self._h))
        _check(_lib.hec_dist_get_info(self._h, ctypes.byref(self.info)))

    def check(self):
        """Synchronise the communication stream; raise if a peer-memory wait timed out."""
        _check(_lib.hec_dist_check(self._h))

    @property
    def handle(self) -> int:
        return self._h.value

    @property
    def n_loc(self) -> int:
        return self.info.r1 - self.info.r0

    def spmv(self, x_local, y_local, stream=None):
        _check(_lib.hec_spmv_dist(self._h, _dptr(x_local, self.n_loc, "x_local"),
                                  _dptr(y_local, self.n_loc, "y_local"), _stream_ptr(stream)))
        return y_local

    def spmv_host(self, x_local, y_local=None, stream=None):
        """COLLECTIVE y_local = (A x)[r0:r1] with HOST buffers (hec_spmv_dist_host):
        H2D of x_local, the distributed product, D2H of y_local; synchronous."""
        if y_local is None:
            y_local = np.empty(self.n_loc, np.float64)
        _check(_lib.hec_spmv_dist_host(self._h, _hptr(x_local, self.n_loc, "x_local"),
                                       _hptr(y_local, self.n_loc, "y_local"), _stream_ptr(stream)))
        return y_local

    def set_timing(self, enable: bool = True):
        """Record phase events in every hec_spmv_dist call (hec_dist_set_timing)."""
        _check(_lib.hec_dist_set_timing(self._h, int(bool(enable))))

    def phase_times(self) -> tuple[float, float]:
        """(interior_ms, comm_ms) of the last timed call, both from its start;
        comm_ms = -1 without an exchange (hec_dist_phase_times)."""
        a, b = ctypes.c_float(), ctypes.c_float()
        _check(_lib.hec_dist_phase_times(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def comm_size(self) -> tuple[int, int]:
        """(ncclCommCount of the handle's communicator or 0, ncclGetVersion)."""
        n, v = i32(), i32()
        _check(_lib.hec_dist_comm_size(self._h, ctypes.byref(n), ctypes.byref(v)))
        return n.value, v.value

    def bicgstab(self, b_local, x_local, tol: float = 1e-8, max_it: int = 1000, stream=None) -> SolveInfoT:
        inf = SolveInfoT()
        _check(_lib.hec_bicgstab_dist(self._h, _dptr(b_local, self.n_loc, "b"), _dptr(x_local, self.n_loc, "x"),
                                      float(tol), int(max_it), _stream_ptr(stream), ctypes.byref(inf)))
        return inf

    def cg(self, b_local, x_local, tol: float = 1e-8, max_it: int = 1000, stream=None) -> SolveInfoT:
        inf = SolveInfoT()
        _check(_lib.hec_cg_dist(self._h, _dptr(b_local, self.n_loc, "b"), _dptr(x_local, self.n_loc, "x"),
                                float(tol), int(max_it), _stream_ptr(stream), ctypes.byref(inf)))
        return inf

    def free(self):
        if self._h and self._h.value:
            _lib.hec_dist_free(self._h)
            self._h = vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class LocalDistGroup:
    """All ranks of a partition emulated on ONE device (hec_dist_create_local):
    same kernels and plan, exchange by device-to-device copies."""

    def __init__(self, A, plan: Plan, device: int = 0, options: OptsT | None = None, p2p: bool = False):
        load()
        args = _CsrArgs(A)
        o = options if options is not None else opts()
        arr = (vp * plan.n_parts)()
        _check(_lib.hec_dist_create_local(args.ref(), plan.handle, ctypes.byref(o), device, arr))
        if p2p:
            st = _lib.hec_dist_p2p_connect_local(arr, plan.n_parts)
            if st != 0:
                for p in range(plan.n_parts):
                    _lib.hec_dist_free(arr[p])
                _check(st)
        self.ranks = [Dist(_handle=arr[p]) for p in range(plan.n_parts)]
        self._arr = arr

    def spmv(self, x_locals, y_locals, stream=None):
        n = len(self.ranks)
        xs = (vp * n)(*[_dptr(x_locals[p], self.ranks[p].n_loc, "x_local") for p in range(n)])
        ys = (vp * n)(*[_dptr(y_locals[p], self.ranks[p].n_loc, "y_local") for p in range(n)])
        _check(_lib.hec_spmv_dist_local(self._arr, n, xs, ys, _stream_ptr(stream)))
        return y_locals

    def _solve(self, fn, b_locals, x_locals, tol, max_it, stream):
        n = len(self.ranks)
        bs = (vp * n)(*[_dptr(b_locals[p], self.ranks[p].n_loc, "b_local") for p in range(n)])
        xs = (vp * n)(*[_dptr(x_locals[p], self.ranks[p].n_loc, "x_local") for p in range(n)])
        inf = SolveInfoT()
        _check(fn(self._arr, n, bs, xs, float(tol), int(max_it), _stream_ptr(stream), ctypes.byref(inf)))
        return inf

    def bicgstab(self, b_locals, x_locals, tol: float = 1e-8, max_it: int = 1000, stream=None) -> SolveInfoT:
        """Alg. 4 over all emulated ranks (hec_bicgstab_dist_local)."""
        return self._solve(_lib.hec_bicgstab_dist_local, b_locals, x_locals, tol, max_it, stream)

    def cg(self, b_locals, x_locals, tol: float = 1e-8, max_it: int = 1000, stream=None) -> SolveInfoT:
        """CG over all emulated ranks (hec_cg_dist_local)."""
        return self._solve(_lib.hec_cg_dist_local, b_locals, x_locals, tol, max_it, stream)

    def free(self):
        for r in self.ranks:
            r.free()


def reorder_rcm(A) -> np.ndarray:
    """Reverse Cuthill-McKee ordering (perm[new] = old) of A's symmetrised pattern."""
    load()
    args = _CsrArgs(A)
    perm = np.empty(A.n_rows, np.int32)
    _check(_lib.hec_reorder_rcm(args.ref(), _p(perm)))
    return perm


def partition_order(A, n_parts: int, method: int = ORDER_MULTILEVEL) -> tuple[np.ndarray, np.ndarray]:
    """(perm, part_ptr): a partitioning order (perm[new] = old, parts contiguous
    in the new order) by level-set recursive bisection or the multilevel
    partitioner (hec_partition_order).  Use with permute() and
    partition(B, n_parts, PART_EXPLICIT, part_ptr)."""
    load()
    args = _CsrArgs(A)
    perm = np.empty(A.n_rows, np.int32)
    pp = np.empty(n_parts + 1, np.int32)
    _check(_lib.hec_partition_order(args.ref(), int(n_parts), int(method), _p(perm), _p(pp)))
    return perm, pp


def permute(A, perm: np.ndarray):
    """B = P A P^T (B[i][j] = A[perm[i]][perm[j]]) as a canonical CSR of A's type."""
    load()
    args = _CsrArgs(A)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    rp = np.empty(A.n_rows + 1, np.int32)
    col = np.empty(args.col.shape[0], np.int32)
    val = np.empty(args.col.shape[0], np.float64)
    _check(_lib.hec_permute(args.ref(), _p(perm), _p(rp), _p(col), _p(val)))
    return type(A)(A.n_rows, A.n_cols, rp, col, val)


def axpby(alpha: float, x, beta: float, y, stream=None):
    """Eq. (3): y = alpha x + beta y (device vectors)."""
    load()
    _check(_lib.hec_axpby(y.numel(), float(alpha), _dptr(x, y.numel(), "x"), float(beta),
                          _dptr(y, y.numel(), "y"), _stream_ptr(stream)))
    return y


def axpbyz(alpha: float, x, beta: float, y, z, stream=None):
    """Eq. (4): z = alpha x + beta y (device vectors)."""
    load()
    n = z.numel()
    _check(_lib.hec_axpbyz(n, float(alpha), _dptr(x, n, "x"), float(beta), _dptr(y, n, "y"),
                           _dptr(z, n, "z"), _stream_ptr(stream)))
    return z


def dot(x, y, stream=None) -> float:
    """Eq. (5): <x, y> (device vectors, host result)."""
    load()
    r = ctypes.c_double()
    _check(_lib.hec_dot(x.numel(), _dptr(x, x.numel(), "x"), _dptr(y, x.numel(), "y"), ctypes.byref(r),
                        _stream_ptr(stream)))
    return r.value


def norm2(x, stream=None) -> float:
    """Eq. (6): ||x||_2 (device vector, host result)."""
    load()
    r = ctypes.c_double()
    _check(_lib.hec_norm2(x.numel(), _dptr(x, x.numel(), "x"), ctypes.byref(r), _stream_ptr(stream)))
    return r.value
