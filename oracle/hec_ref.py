"""O2 -- HEC reference builder (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

HEC = an ELL part stored column by column plus the irregular remainder in CSR
(§2.1, "another hybrid format called HEC which saved the
irregular part in a CSR format"; P:73 column-major storage, stride a multiple
of 32, "we set it as 256", ELL/CSR boundary "a recommended value 20").

Readings (restated in DESIGN.md §3):
  A1  width policy BG3 (default): w = min(cap, k*), k* = smallest k >= 0 with
      3 * #{rows: len > k} < n_rows (the Bell-Garland one-third rule the
      citation \\cite{nv-spmv2} points to).  CAP: w = min(cap, max_len)
      (SPEC S:53).  FIXED: w = fixed_width.
  A2  stride s = roundup(n_rows, stride_unit), stride_unit default 256.
  A3  ELL holds the first min(len_i, w) entries of row i in column order.
  A4  padding slot = (col -1, val +0.0).
  A15 the CSR part is compact: only rows that spill, ascending.
Built step by step with plain loops over rows so it can be read against the
definition; numpy only for array storage.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

POLICY_BG3, POLICY_CAP, POLICY_FIXED = 0, 1, 2
SENTINEL = -1


@dataclass
class HecRef:
    n_rows: int
    n_cols: int
    width: int
    stride: int
    ell_col: np.ndarray   # int32[width*stride], column-major: slot j of row i at j*stride + i
    ell_val: np.ndarray   # float64[width*stride]
    tail_rows: np.ndarray  # int32[t_r], ascending
    tail_ptr: np.ndarray   # int32[t_r+1]
    tail_col: np.ndarray   # int32[t_z]
    tail_val: np.ndarray   # float64[t_z]


def row_lengths(A) -> np.ndarray:
    return np.diff(np.asarray(A.row_ptr, dtype=np.int64))


def width_bg3(lengths: np.ndarray, cap: int) -> int:
    """A1: k* = smallest k >= 0 with 3 * #{rows with len > k} < n; w = min(cap, k*)."""
    n = len(lengths)
    if n == 0:
        return 0
    k = 0
    while True:
        longer = int(np.count_nonzero(lengths > k))
        if 3 * longer < n:
            break
        k += 1
    return min(cap, k)


def width_cap(lengths: np.ndarray, cap: int) -> int:
    """ell_width = min(cap, max row nnz)."""
    return min(cap, int(lengths.max()) if len(lengths) else 0)


def choose_width(lengths: np.ndarray, policy: int = POLICY_BG3, cap: int = 20,
                 fixed_width: int = 0) -> int:
    if policy == POLICY_BG3:
        return width_bg3(lengths, cap)
    if policy == POLICY_CAP:
        return width_cap(lengths, cap)
    if policy == POLICY_FIXED:
        return fixed_width
    raise ValueError("unknown width policy")


def stride_for(n_rows: int, stride_unit: int = 256) -> int:
    """A2: s = roundup(n_rows, stride_unit) (P:73 'a multiple of 32 ... 256')."""
    return ((n_rows + stride_unit - 1) // stride_unit) * stride_unit


def build(A, policy: int = POLICY_BG3, cap: int = 20, fixed_width: int = 0,
          stride_unit: int = 256, width: int | None = None) -> HecRef:
    """CSR -> HEC.  ``width`` overrides the policy (used for distributed
    sub-matrices that inherit their partition's width, reading A12)."""
    lengths = row_lengths(A)
    w = choose_width(lengths, policy, cap, fixed_width) if width is None else width
    s = stride_for(A.n_rows, stride_unit)
    ell_col = np.full(w * s, SENTINEL, dtype=np.int32)
    ell_val = np.zeros(w * s, dtype=np.float64)
    tail_rows, tail_ptr, tail_col, tail_val = [], [0], [], []
    rp = np.asarray(A.row_ptr, dtype=np.int64)
    for i in range(A.n_rows):
        b, e = int(rp[i]), int(rp[i + 1])
        m = min(e - b, w)
        for j in range(m):                       # A3: first min(len, w) entries -> ELL
            ell_col[j * s + i] = A.col[b + j]
            ell_val[j * s + i] = A.val[b + j]
        if e - b > w:                            # A15: the rest, in order -> tail
            tail_rows.append(i)
            tail_col.extend(A.col[b + w:e])
            tail_val.extend(A.val[b + w:e])
            tail_ptr.append(len(tail_col))
    return HecRef(A.n_rows, A.n_cols, w, s, ell_col, ell_val,
                  np.array(tail_rows, np.int32), np.array(tail_ptr, np.int32),
                  np.array(tail_col, np.int32), np.array(tail_val, np.float64))


def build_fast(A, policy: int = POLICY_BG3, cap: int = 20, fixed_width: int = 0,
               stride_unit: int = 256, width: int | None = None) -> HecRef:
    """Same construction as ``build`` with the row loop vectorised (for the
    multi-million-row configs).  tests/test_oracle_hec.py checks that it equals
    ``build`` on every small case."""
    lengths = row_lengths(A)
    w = choose_width(lengths, policy, cap, fixed_width) if width is None else width
    s = stride_for(A.n_rows, stride_unit)
    n = A.n_rows
    rp = np.asarray(A.row_ptr, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), lengths)
    slot = np.arange(len(A.col), dtype=np.int64) - rp[rows]
    in_ell = slot < w
    ell_col = np.full(w * s, SENTINEL, dtype=np.int32)
    ell_val = np.zeros(w * s, dtype=np.float64)
    pos = slot[in_ell] * s + rows[in_ell]
    ell_col[pos] = A.col[in_ell]
    ell_val[pos] = A.val[in_ell]
    spill = lengths > w
    tail_rows = np.nonzero(spill)[0].astype(np.int32)
    tail_ptr = np.zeros(len(tail_rows) + 1, np.int64)
    tail_ptr[1:] = np.cumsum(lengths[spill] - w)
    return HecRef(n, A.n_cols, w, s, ell_col, ell_val, tail_rows, tail_ptr.astype(np.int32),
                  np.ascontiguousarray(A.col[~in_ell], dtype=np.int32),
                  np.ascontiguousarray(A.val[~in_ell], dtype=np.float64))


def reconstruct(H: HecRef):
    """Inverse map HEC -> per-row (col, val) lists (round-trip invariant)."""
    rows = [[] for _ in range(H.n_rows)]
    for i in range(H.n_rows):
        for j in range(H.width):
            c = int(H.ell_col[j * H.stride + i])
            if c != SENTINEL:
                rows[i].append((c, float(H.ell_val[j * H.stride + i])))
    for t, r in enumerate(H.tail_rows):
        for k in range(int(H.tail_ptr[t]), int(H.tail_ptr[t + 1])):
            rows[int(r)].append((int(H.tail_col[k]), float(H.tail_val[k])))
    return rows


def spmv(H: HecRef, x: np.ndarray) -> np.ndarray:
    """Alg. 1 literally: ELL loop over all rows first, then the
    CSR loop; each row a sequential sum.  Reference for the HEC *evaluation
    order*, used only to pin reconstruct/spmv consistency on small inputs."""
    y = np.zeros(H.n_rows, dtype=np.float64)
    for i in range(H.n_rows):                   # "for i = 1:n  (ELL)"
        s = 0.0
        for j in range(H.width):
            c = int(H.ell_col[j * H.stride + i])
            if c != SENTINEL:
                s = s + float(H.ell_val[j * H.stride + i]) * float(x[c])
        y[i] = s
    for t, r in enumerate(H.tail_rows):         # "for i = 1:n  (CSR)"
        s = 0.0
        for k in range(int(H.tail_ptr[t]), int(H.tail_ptr[t + 1])):
            s = s + float(H.tail_val[k]) * float(x[int(H.tail_col[k])])
        y[int(r)] = y[int(r)] + s
    return y
