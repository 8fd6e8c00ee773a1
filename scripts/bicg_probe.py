"""BiCGSTAB iteration count on the power-law 20000 test matrix (GPU) -- run
under different env knobs to see which part of the SpMV changes it."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import hecgen, paper_1606_00545_b200 as hec
A = hecgen.powerlaw(20000, seed=3)
b = hecgen.vector(A.n_rows, "uniform", seed=12)
M = hec.from_csr(A)
out = {}
for it in range(3):
    xd = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
    info = M.bicgstab(torch.from_numpy(b).cuda(), xd, 1e-10, 2000)
    out[f"run{it}"] = [info.iterations, info.rel_residual]
x = hecgen.vector(A.n_cols, "uniform", seed=5)
yd = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
M.spmv(torch.from_numpy(x).cuda(), yd)
out["y_sum"] = float(yd.sum())
out["env"] = {k: v for k, v in os.environ.items() if k.startswith("HEC_")}
print(json.dumps(out))
