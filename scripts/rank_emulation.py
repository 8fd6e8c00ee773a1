"""Compute-only projection of the row-partitioned SpMV on ONE GPU (this run
has a single B200): for P = 1, 2, 4, 8 every part's local matrix
(its rows; owned columns renumbered to [0, n_loc), halo columns to
n_loc + rank in the sorted halo set, DESIGN reading A10; width from the part's
own histogram, A12) is built as a standalone HEC and timed alone with
hec_spmv.  T_proj(P) = max over parts -- the critical path if the halo
exchange is fully hidden behind the interior rows (the design's overlap) --
and E_proj(P) = T(1) / (P T_proj(P)).  It isolates the compute imbalance the
partition leaves (ELL/tail split, nnz balance); it does not measure NVLink.

  python scripts/rank_emulation.py powerlaw_8M_dsorted [--parts 1 2 4 8] [--reps 30]
Prints one JSON line per config.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import hecgen
import paper_1606_00545_b200 as hec


def local_csr(A, r0, r1):
    rp = A.row_ptr
    b, e = int(rp[r0]), int(rp[r1])
    cols = A.col[b:e]
    own = (cols >= r0) & (cols < r1)
    halo = np.unique(cols[~own])
    n_loc = r1 - r0
    lc = np.where(own, cols - r0, n_loc + np.searchsorted(halo, cols)).astype(np.int32)
    val = np.ascontiguousarray(A.val[b:e])
    if len(halo):
        # canonical local order per row: owned columns, then halo columns below
        # r0, then above r1 (each run already ascending)
        cls = np.where(own, 0, np.where(cols < r0, 1, 2)).astype(np.int64)
        row = np.repeat(np.arange(n_loc, dtype=np.int64), np.diff(rp[r0:r1 + 1]))
        o = np.argsort(row * 3 + cls, kind="stable")
        lc, val = lc[o], val[o]
    return hecgen.Csr(n_loc, n_loc + len(halo), (rp[r0:r1 + 1] - b).astype(np.int32), lc, val,
                      name=f"{A.name}[{r0}:{r1})"), len(halo)


def time_spmv(M, n_cols, n_rows, reps, flush):
    x = torch.from_numpy(hecgen.vector(n_cols, "uniform", seed=1606)).cuda()
    y = torch.empty(n_rows, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    fl = bench.L2Flusher("cuda") if flush else None
    with torch.cuda.stream(s):
        for _ in range(5):
            M.spmv(x, y, s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(s):
            if fl:
                fl()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            M.spmv(x, y, s)
            b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--parts", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--kind", choices=["auto", "nnz", "cost"], default="auto",
                    help="partition of non-grid matrices: CONTIG_NNZ (auto) or CONTIG_COST")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for cfg in args.configs:
        A = hecgen.CONFIGS[cfg]()
        kind = (hec.PART_GRID if A.grid is not None else
                hec.PART_CONTIG_COST if args.kind == "cost" else hec.PART_CONTIG_NNZ)
        kname = {hec.PART_GRID: "GRID", hec.PART_CONTIG_NNZ: "CONTIG_NNZ", hec.PART_CONTIG_COST: "CONTIG_COST"}[kind]
        out = {"config": cfg, "n_rows": A.n_rows, "nnz": A.nnz, "partition": kname,
               "what": "compute-only projection on one GPU: each part's local HEC timed alone (median of reps, "
                       "L2 flushed when the part is < 4x L2); T_proj = max over parts", "P": {}}
        t1 = None
        for P in args.parts:
            plan = hec.partition(A, P, kind, A.grid)
            pp = plan.part_ptr()
            parts = []
            for p in range(P):
                r0, r1 = int(pp[p]), int(pp[p + 1])
                L, n_halo = local_csr(A, r0, r1)
                M = hec.from_csr(L)
                alg = 12 * L.nnz + 8 * L.n_cols + 8 * L.n_rows
                t = time_spmv(M, L.n_cols, L.n_rows, args.reps, alg < 4 * bench.L2_BYTES)
                i = M.info
                parts.append({"rows": L.n_rows, "nnz": L.nnz, "halo": n_halo, "width": i.ell_width,
                              "tail_nnz_frac": round(i.tail_nnz / max(1, L.nnz), 4), "ms": round(t, 5),
                              "gbs": round(alg / (t * 1e-3) / 1e9, 1)})
                M.free()
                del L
            tp = max(q["ms"] for q in parts)
            if P == 1:
                t1 = tp
            rec = {"T_proj_ms": tp, "parts": parts}
            if t1:
                rec["E_proj"] = round(t1 / (P * tp), 4)
            out["P"][P] = rec
            print(f"{cfg} [{kname}] P={P}: T_proj {tp:.4f} ms" + (f", E_proj {rec['E_proj']}" if t1 else ""), file=sys.stderr)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
