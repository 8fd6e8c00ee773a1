"""The event-timed cold-launch floor of bench.py's protocol on this box: the
same L2 flush, then an event pair around ONE trivial kernel (a 1-element
fill) -- what every cold single-launch measurement pays before its bytes."""
import json, statistics, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import L2Flusher
torch.cuda.set_device(0)
fl = L2Flusher("cuda:0")
t = torch.zeros(1, dtype=torch.float64, device="cuda")
for _ in range(10):
    fl(); t.fill_(1.0)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
for a, b in ev:
    fl()
    a.record()
    t.fill_(2.0)
    b.record()
torch.cuda.synchronize()
per = [a.elapsed_time(b) * 1e3 for a, b in ev]
print(json.dumps({"what": "event pair around one 1-element fill kernel after the bench L2 flush",
                  "median_us": round(statistics.median(per), 2), "p10_us": round(sorted(per)[20], 2),
                  "mean_us": round(statistics.mean(per), 2)}))
