"""O3 / O4 -- partition, halo plan and distributed-result references
(TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md §2.2: the rows are partitioned ("sequence partition" for
FDM/FVM matrices, METIS otherwise), the vector is split into segments
conformally, and each GPU receives the x entries that "a segment vector can not
provide" through a shared cache.  Readings:
  A9  GRID: part p owns planes [floor(p*nz/P), floor((p+1)*nz/P)) of the slowest
      axis with extent > 1; CONTIG_ROWS: floor(p*n/P); CONTIG_NNZ:
      lower_bound(row_ptr, ceil(p*nnz/P)) then clamped so every part is
      non-empty.  The row permutation is the identity.  CONTIG_COST (ours,
      DESIGN.md §6): CONTIG_NNZ re-balanced on a padded-slots + tail-entries
      cost under each part's own width.
  A10 recv_p sorted ascending by global column (hence grouped by owner);
      local column of halo entry g = n_loc + rank of g in recv_p; send lists
      are sorted local indices, concatenated over peers in rank order.
  A11 boundary row = a row with >= 1 stored column outside its part.
  A12 the partition's width is chosen from the histogram of all its local
      rows; interior and boundary sub-HECs inherit it.
Every set is computed from its definition with plain Python loops/sets.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

KIND_CONTIG_NNZ, KIND_CONTIG_ROWS, KIND_GRID, KIND_CONTIG_COST = 0, 1, 2, 3


def part_ptr_ref(A, n_parts: int, kind: int = KIND_CONTIG_NNZ, grid=None) -> np.ndarray:
    n = A.n_rows
    if n_parts < 1 or n_parts > n:
        raise ValueError("n_parts out of range")
    pp = [0] * (n_parts + 1)
    pp[n_parts] = n
    if kind == KIND_CONTIG_ROWS:
        for p in range(1, n_parts):
            pp[p] = (p * n) // n_parts
    elif kind == KIND_GRID:
        nx, ny, nz = grid
        if nx * ny * nz != n:
            raise ValueError("grid does not match n")
        if nz > 1:
            ext, plane = nz, nx * ny
        elif ny > 1:
            ext, plane = ny, nx
        else:
            ext, plane = nx, 1
        if n_parts > ext:
            raise ValueError("more parts than planes")
        for p in range(1, n_parts):
            pp[p] = ((p * ext) // n_parts) * plane
    elif kind == KIND_CONTIG_NNZ:
        rp = [int(v) for v in A.row_ptr]
        nnz = rp[-1]
        for p in range(1, n_parts):
            t = -((-p * nnz) // n_parts)            # ceil(p*nnz/P)
            r = 0
            while r < n and rp[r] < t:              # lower_bound(row_ptr, t)
                r += 1
            r = max(r, pp[p - 1] + 1)
            r = min(r, n - (n_parts - p))
            pp[p] = r
    elif kind == KIND_CONTIG_COST:
        # not in the paper: modeled-cost balance.  Start from
        # CONTIG_NNZ; then (at most 4 times, stopping at a fixed point) give row
        # i of part p the cost 3 w_p + 4 max(len_i - w_p, 0), w_p = the BG3
        # width (A1, cap 20) of part p's rows, and cut where the prefix cost
        # first reaches ceil(p C / P), clamped as for CONTIG_NNZ.
        from .hec_ref import width_bg3
        lens = [int(A.row_ptr[i + 1]) - int(A.row_ptr[i]) for i in range(n)]
        cur = [int(v) for v in part_ptr_ref(A, n_parts, KIND_CONTIG_NNZ)]
        for _ in range(4):
            cost = []
            for p in range(n_parts):
                w = width_bg3(np.array(lens[cur[p]:cur[p + 1]], dtype=np.int64), 20)
                for i in range(cur[p], cur[p + 1]):
                    cost.append(3 * w + 4 * max(lens[i] - w, 0))
            prefix = [0]
            for c in cost:
                prefix.append(prefix[-1] + c)
            C = prefix[-1]
            nxt = [0] * (n_parts + 1)
            nxt[n_parts] = n
            for p in range(1, n_parts):
                t = -((-p * C) // n_parts)           # ceil(p*C/P)
                r = 0
                while r < n and prefix[r] < t:      # lower_bound(prefix, t)
                    r += 1
                r = max(r, nxt[p - 1] + 1)
                r = min(r, n - (n_parts - p))
                nxt[p] = r
            if nxt == cur:
                break
            cur = nxt
        pp = cur
    else:
        raise ValueError("unknown partition kind")
    return np.array(pp, dtype=np.int32)


@dataclass
class PartRef:
    r0: int
    r1: int
    recv: np.ndarray        # int32 global columns, ascending
    recv_off: np.ndarray    # int32[P+1]: recv from peer q is recv[recv_off[q]:recv_off[q+1]]
    send_idx: np.ndarray    # int32 local indices, concatenated over peers ascending
    send_off: np.ndarray    # int32[P+1]
    interior: np.ndarray    # int32 local row ids
    boundary: np.ndarray    # int32 local row ids
    local_rows: list = field(default_factory=list)  # per local row: [(local col, val)]

    @property
    def n_loc(self) -> int:
        return self.r1 - self.r0


def owner_of(part_ptr: np.ndarray, j: int) -> int:
    q = 0
    while not (part_ptr[q] <= j < part_ptr[q + 1]):
        q += 1
    return q


def plan_ref(A, part_ptr: np.ndarray) -> list[PartRef]:
    P = len(part_ptr) - 1
    rp = A.row_ptr
    recvs = []
    for p in range(P):
        r0, r1 = int(part_ptr[p]), int(part_ptr[p + 1])
        s = set()
        for i in range(r0, r1):
            for k in range(int(rp[i]), int(rp[i + 1])):
                j = int(A.col[k])
                if not (r0 <= j < r1):
                    s.add(j)
        recvs.append(sorted(s))
    parts = []
    for p in range(P):
        r0, r1 = int(part_ptr[p]), int(part_ptr[p + 1])
        recv = recvs[p]
        recv_off = [0] * (P + 1)
        for q in range(P):
            recv_off[q + 1] = recv_off[q] + sum(1 for j in recv if owner_of(part_ptr, j) == q)
        send, send_off = [], [0]
        for q in range(P):
            lst = sorted(j - r0 for j in recvs[q] if r0 <= j < r1) if q != p else []
            send.extend(lst)
            send_off.append(len(send))
        pos = {j: t for t, j in enumerate(recv)}
        interior, boundary, local_rows = [], [], []
        for i in range(r0, r1):
            row = []
            outside = False
            for k in range(int(rp[i]), int(rp[i + 1])):
                j = int(A.col[k])
                if r0 <= j < r1:
                    row.append((j - r0, float(A.val[k])))
                else:
                    outside = True
                    row.append(((r1 - r0) + pos[j], float(A.val[k])))
            local_rows.append(row)
            (boundary if outside else interior).append(i - r0)
        parts.append(PartRef(r0, r1, np.array(recv, np.int32), np.array(recv_off, np.int32),
                             np.array(send, np.int32), np.array(send_off, np.int32),
                             np.array(interior, np.int32), np.array(boundary, np.int32),
                             local_rows))
    return parts


def local_csr(part: PartRef, which: str, csr_type):
    """Local sub-matrix of a part: 'interior', 'boundary' or 'all' rows, with
    local column numbering (owned -> [0,n_loc), halo -> n_loc + pos).  Each
    row is re-sorted by LOCAL column id (reading A3 applied to the local
    matrix: a halo column numbered n_loc+pos sorts after every owned one)."""
    rows = {"interior": part.interior, "boundary": part.boundary,
            "all": np.arange(part.n_loc, dtype=np.int32)}[which]
    rp, col, val = [0], [], []
    for i in rows:
        row = sorted(part.local_rows[int(i)])
        col.extend(c for c, _ in row)
        val.extend(v for _, v in row)
        rp.append(len(col))
    n_cols = part.n_loc + len(part.recv)
    return csr_type(len(rows), n_cols, np.array(rp, np.int32), np.array(col, np.int32),
                    np.array(val, np.float64))


def part_width(part: PartRef, csr_type, policy: int = 0, cap: int = 20, fixed_width: int = 0) -> int:
    """A12: the partition's ELL width from the histogram of ALL its local rows."""
    from .hec_ref import choose_width, row_lengths
    return choose_width(row_lengths(local_csr(part, "all", csr_type)), policy, cap, fixed_width)


def simulated_dist_spmv(A, part_ptr: np.ndarray, parts: list[PartRef], x: np.ndarray,
                        spmv_fn, csr_type) -> np.ndarray:
    """O4 with an explicit exchange: each part builds x_ext = [x_loc | x_halo],
    where x_halo is filled ONLY through the peers' send lists (the paper's
    shared cache), then multiplies its local rows.  Equals O1 on the
    whole matrix iff the plan is complete."""
    P = len(parts)
    cache = {}
    for q in range(P):                               # export to the cache
        xq = x[parts[q].r0:parts[q].r1]
        for p in range(P):
            lo, hi = int(parts[q].send_off[p]), int(parts[q].send_off[p + 1])
            cache[(q, p)] = xq[parts[q].send_idx[lo:hi]]
    y = np.empty(A.n_rows, dtype=np.float64)
    for p in range(P):                               # import from the cache
        part = parts[p]
        halo = np.empty(len(part.recv), dtype=np.float64)
        for q in range(P):
            lo, hi = int(part.recv_off[q]), int(part.recv_off[q + 1])
            halo[lo:hi] = cache[(q, p)]
        x_ext = np.concatenate([x[part.r0:part.r1], halo])
        L = local_csr(part, "all", csr_type)
        y[part.r0:part.r1] = spmv_fn(L, x_ext)
    return y
