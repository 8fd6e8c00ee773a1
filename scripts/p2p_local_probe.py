"""Local emulation of the 8-slab 256^3 partition through the peer-memory
transport: runs a few hec_spmv_dist_local calls (for an ncu launch list of
push_kernel / peer_wait_kernel / interior / boundary kernels on one GPU)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import hecgen
import paper_1606_00545_b200 as hec

A = hecgen.poisson3d(256, 256, 256)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
plan = hec.partition(A, P, hec.PART_GRID, (256, 256, 256))
grp = hec.LocalDistGroup(A, plan, 0, None, p2p=True)
pp = plan.part_ptr()
x = hecgen.vector(A.n_cols, "uniform", seed=1606)
xs = [torch.from_numpy(np.ascontiguousarray(x[pp[p]:pp[p + 1]])).cuda() for p in range(P)]
ys = [torch.empty(int(pp[p + 1] - pp[p]), dtype=torch.float64, device="cuda") for p in range(P)]
for _ in range(4):
    grp.spmv(xs, ys)
torch.cuda.synchronize()
for r in grp.ranks:
    r.check()
print("ok", [r.info.launches for r in grp.ranks], [r.info.n_send for r in grp.ranks])
