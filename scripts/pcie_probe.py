"""Measure pinned H2D / D2H / concurrent copy bandwidth (context for the e2e number)."""
import json, time, torch
n = 16 * 1024 * 1024
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
r = {"bytes": 8 * n, "h2d_ms": t(h2d) * 1e3, "d2h_ms": t(d2h) * 1e3, "both_ms": t(both) * 1e3}
r.update({k.replace("_ms", "_GBs"): round(8 * n / (v * 1e-3) / 1e9, 1) for k, v in list(r.items()) if k.endswith("_ms")})
print(json.dumps(r))
