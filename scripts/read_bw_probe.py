"""Read-bandwidth ceiling probe: torch reductions / copies over ~1.6 GB, CUDA
events, best of 20 -- the context for ell_kernel's 6.79 TB/s on 256^3."""
import json
import torch
n = 1_673_003_008 // 8
a = torch.ones(n, dtype=torch.float64, device="cuda")
b = torch.empty(n // 12, dtype=torch.float64, device="cuda")
def best(fn, k=20):
    ts = []
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
out = {}
t = best(lambda: a.sum()); out["sum_read_GBs"] = round(8 * n / t / 1e6, 1)
t = best(lambda: torch.max(a)); out["max_read_GBs"] = round(8 * n / t / 1e6, 1)
c = a[: n // 2]; d = torch.empty_like(c)
t = best(lambda: d.copy_(c)); out["copy_rw_GBs"] = round(2 * 8 * (n // 2) / t / 1e6, 1)
print(json.dumps(out))
