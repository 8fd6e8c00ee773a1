"""Summarise a gpu_ring.sh run: step ms / frac (bench) and, per kernel, ncu us, DRAM GB and
L1 global-load sectors (M) of the last profiled step."""
import csv
import glob
import json
import os
import sys

d = sys.argv[1]
for b in sorted(glob.glob(os.path.join(d, "b_*.json"))):
    name = os.path.basename(b)[2:-5]
    try:
        j = json.loads(open(b).read().strip().splitlines()[-1])
        ms, frac = j["ms_per_step"], j["roofline"]["frac"]
    except Exception:
        ms = frac = None
    per = {}
    lf = os.path.join(d, f"l_{name}.csv")
    if os.path.exists(lf):
        rows = list(csv.reader(ln for ln in open(lf) if ln.startswith('"')))
        if rows:
            h = rows[0]
            for r in rows[1:]:
                k = r[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").replace("hec::", "")
                m, v = r[h.index("Metric Name")], float(r[h.index("Metric Value")].replace(",", ""))
                per.setdefault(k, {})[m] = v  # last launch of each kernel wins
    ks = "  ".join(f"{k} {v.get('gpu__time_duration.sum', 0) / 1e3:.1f}us "
                   f"{v.get('dram__bytes_read.sum', 0) / 1e9:.3f}GB "
                   f"w{v.get('dram__bytes_write.sum', 0) / 1e9:.3f}GB "
                   f"{v.get('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 0) / 1e6:.1f}Ms"
                   for k, v in sorted(per.items()))
    print(f"{name:22s} step {ms} ms frac {frac}   {ks}")
