"""GPU BiCGSTAB relative residual after k iterations on the power-law 20000
test matrix (compare with the oracle's history on the host)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import hecgen, paper_1606_00545_b200 as hec
A = hecgen.powerlaw(20000, seed=3)
b = hecgen.vector(A.n_rows, "uniform", seed=12)
M = hec.from_csr(A)
out = {}
for k in (1, 5, 10, 20, 40, 60, 80, 100, 120, 140, 160, 180):
    xd = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
    info = M.bicgstab(torch.from_numpy(b).cuda(), xd, 1e-30, k)
    out[k] = info.rel_residual
print(json.dumps(out))
