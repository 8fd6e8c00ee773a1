import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, hecgen
import paper_1606_00545_b200 as hec
A = hecgen.poisson3d(256, 256, 256)
M = hec.from_csr(A)
b = torch.from_numpy(hecgen.vector(A.n_rows, "uniform", seed=7)).cuda()
x = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
for solver in ("cg", "bicgstab"):
    f = getattr(M, solver)
    f(b, x, 0.0, 3); torch.cuda.synchronize()
    for K in (10, 50, 100):
        x.zero_(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); info = f(b, x, 0.0, K); e1.record(); torch.cuda.synchronize()
        print(solver, K, info.iterations, round(e0.elapsed_time(e1) / info.iterations, 4), "ms/it (events)",
              round((time.perf_counter() - t0) * 1e3 / info.iterations, 4), "ms/it (wall)", flush=True)
