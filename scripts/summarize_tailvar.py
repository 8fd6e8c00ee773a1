"""Summarise a gpu_tailvar.sh run: step ms (bench) and tail kernel us / DRAM GB (ncu)."""
import csv, glob, json, os, sys
d = sys.argv[1]
for b in sorted(glob.glob(os.path.join(d, "b_*.json"))):
    name = os.path.basename(b)[2:-5]
    try:
        j = json.loads(open(b).read().strip().splitlines()[-1])
        ms = j["ms_per_step"]
    except Exception:
        ms = None
    t, dr = [], []
    lf = os.path.join(d, f"l_{name}.csv")
    if os.path.exists(lf):
        rows = list(csv.reader(l for l in open(lf) if l.startswith('"')))
        if rows:
            h = rows[0]
            for r in rows[1:]:
                if r[h.index("Metric Name")] == "gpu__time_duration.sum":
                    t.append(float(r[h.index("Metric Value")]) / 1e3)
                if r[h.index("Metric Name")] == "dram__bytes_read.sum":
                    dr.append(float(r[h.index("Metric Value")]) / 1e9)
    print(f"{name:24s} step {ms} ms   tail {min(t) if t else None} us   dram {dr[-1] if dr else None} GB")
