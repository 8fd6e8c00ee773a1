"""Per-step time series of hec_spmv on one config (event pair per step, no flush for inputs > 4x L2),
with the SM clock and throttle reasons sampled beside it: are slow steps periodic, clustered in time,
or tied to a setting?  Usage: python scripts/step_series.py CONFIG STEPS [ENV=VAL ...] (env applied
before the handle is built)."""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for kv in sys.argv[3:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hecgen  # noqa: E402
import paper_1606_00545_b200 as hec  # noqa: E402

cfg, K = sys.argv[1], int(sys.argv[2])
A = hecgen.CONFIGS[cfg]()
x = torch.from_numpy(hecgen.vector(A.n_cols, "uniform", seed=1606)).cuda()
y = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
M = hec.from_csr(A)
s = torch.cuda.Stream()
for _ in range(20):
    M.spmv(x, y, s)
torch.cuda.synchronize()
clk = []
stop = False


def sample():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    t0 = time.perf_counter()
    while not stop:
        clk.append((time.perf_counter() - t0, pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h), pynvml.nvmlDeviceGetPowerUsage(h)))
        time.sleep(0.002)


th = threading.Thread(target=sample)
th.start()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
with torch.cuda.stream(s):
    for k in range(K):
        ev[k][0].record(s)
        M.spmv(x, y, s)
        ev[k][1].record(s)
torch.cuda.synchronize()
stop = True
th.join()
t = [a.elapsed_time(b) for a, b in ev]
print(json.dumps({"config": cfg, "env": sys.argv[3:], "ms": [round(v, 5) for v in t],
                  "median": float(np.median(t)), "mean": float(np.mean(t)),
                  "clock_samples": [(round(a, 4), c, int(r), p) for a, c, r, p in clk]}))
