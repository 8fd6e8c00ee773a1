"""Probe: how the x-gather DRAM refetch of the power-law SpMV grows with n
(x = 8n bytes vs the 126 MB L2).  Run under ncu with dram__bytes_read.sum."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import hecgen
import paper_1606_00545_b200 as hec

for lg in [int(a) for a in sys.argv[1:]]:
    A = hecgen.powerlaw(1 << lg)
    M = hec.from_csr(A)
    x = torch.from_numpy(hecgen.vector(A.n_cols, "uniform", seed=1)).cuda()
    y = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
    for _ in range(3):
        M.spmv(x, y)
    torch.cuda.synchronize()
    inf = M.info
    print(f"lg {lg} n {A.n_rows} nnz {A.nnz} x_MB {8*A.n_cols/1e6:.1f} ell_bytes {12*inf.ell_width*inf.ell_stride} "
          f"tail_bytes {12*inf.tail_nnz + 8*inf.tail_rows}", flush=True)
    M.free()
