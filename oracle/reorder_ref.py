"""Reordering reference (NEXT-4) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §2.2: for irregular matrices "the rows of the matrix are
switched first and all the nonzero entries are put along the diagonal as close
as possible".  METIS is not available offline; the reading (A21) is
reverse Cuthill-McKee on the pattern of A + A^T, written here step by step
with plain Python lists:

  for each connected component, in order of its lowest vertex:
    start = the component's lowest-(degree, index) vertex; depth = -1
    repeat: BFS from start -> last level L and eccentricity d;
            cand = lowest-(degree, index) vertex of L;
            stop if d <= depth or cand == start; else depth = d, start = cand
    Cuthill-McKee BFS from start, appending each vertex's unvisited
    neighbours in increasing (degree, index) order
  reverse the whole sequence;  perm[new] = old.

permute(A, perm) is the plain definition B[i][j] = A[perm[i]][perm[j]].
"""
from __future__ import annotations

import numpy as np


def adjacency(A) -> list[list[int]]:
    n = A.n_rows
    nb = [set() for _ in range(n)]
    for i in range(n):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            j = int(A.col[k])
            if j != i:
                nb[i].add(j)
                nb[j].add(i)
    return [sorted(s) for s in nb]


def rcm(A) -> np.ndarray:
    n = A.n_rows
    adj = adjacency(A)
    deg = [len(a) for a in adj]
    key = lambda v: (deg[v], v)  # noqa: E731
    done = [False] * n
    order = []
    for seed in range(n):
        if done[seed]:
            continue
        comp, seen = [seed], {seed}
        for v in comp:
            for u in adj[v]:
                if u not in seen:
                    seen.add(u)
                    comp.append(u)
        start = min(comp, key=key)
        depth = -1
        while True:
            level, visited, d = [start], {start}, 0
            while True:
                nxt = []
                for v in level:
                    for u in adj[v]:
                        if not done[u] and u not in visited:
                            visited.add(u)
                            nxt.append(u)
                if not nxt:
                    break
                level, d = nxt, d + 1
            cand = min(level, key=key)
            if d <= depth or cand == start:
                break
            depth, start = d, cand
        base = len(order)
        order.append(start)
        done[start] = True
        h = base
        while h < len(order):
            v = order[h]
            for u in sorted((u for u in adj[v] if not done[u]), key=key):
                done[u] = True
                order.append(u)
            h += 1
    return np.array(order[::-1], dtype=np.int32)


def permute(A, perm: np.ndarray, csr_type):
    n = A.n_rows
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    rp, col, val = [0], [], []
    for i in range(n):
        o = int(perm[i])
        row = sorted((int(inv[A.col[k]]), float(A.val[k])) for k in range(A.row_ptr[o], A.row_ptr[o + 1]))
        col.extend(c for c, _ in row)
        val.extend(v for _, v in row)
        rp.append(len(col))
    return csr_type(n, n, np.array(rp, np.int32), np.array(col, np.int32), np.array(val, np.float64))


def bandwidth(A) -> int:
    b = 0
    for i in range(A.n_rows):
        for k in range(A.row_ptr[i], A.row_ptr[i + 1]):
            b = max(b, abs(int(A.col[k]) - i))
    return b
