#!/usr/bin/env python
"""Summarise an ncu --set full report (read here, no GPU needed) into a small
text table + JSON, for committing under profiles/.

  python scripts/ncu_summary.py gpurun_out/r01/prof_ell.ncu-rep profiles/r01/ncu_ell_full.txt [--config poisson3d_256]
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
    "l1tex__t_sector_hit_rate.pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__grid_size",
    "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * mult.get(unit, 1)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    config = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines, launches = [], []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        d = {"kernel": name}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = (r[i], units[i])
        rd = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
        wr = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
        d["dram_bytes_per_launch"] = (rd + wr) if rd is not None and wr is not None else None
        launches.append(d)
        lines.append(f"== {name}")
        for m in METRICS:
            if m in d:
                lines.append(f"  {m:60s} {d[m][0]:>16s} {d[m][1]}")
        if d["dram_bytes_per_launch"]:
            lines.append(f"  {'dram read+write per launch (bytes)':60s} {d['dram_bytes_per_launch']:16.0f}")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary of {os.path.basename(rep)}\n")
        f.write("\n".join(lines) + "\n")
    if config and launches:
        tj = os.path.join(os.path.dirname(os.path.dirname(out)), "ncu_traffic.json")
        try:
            cur = json.load(open(tj))
        except Exception:
            cur = {}
        vals = [l["dram_bytes_per_launch"] for l in launches if l["dram_bytes_per_launch"]]
        ent = cur.get(config, {})
        kern = ent.get("kernels", {})
        kname = launches[0]["kernel"].split("(")[0].replace("void ", "")
        kern[kname.split("<")[0]] = {"dram_bytes_per_launch": round(sum(vals) / len(vals)), "kernel": kname,
                                     "source": os.path.relpath(out, os.path.dirname(tj))}
        # a step launches each of these kernels once: its traffic is their sum
        # keyed by the native sources the capture was taken with: bench.py
        # reports it only while csrc/ + include/ still hash to this value
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from bench import csrc_hash
        ent = {"dram_bytes_per_step": sum(k["dram_bytes_per_launch"] for k in kern.values()), "kernels": kern,
               "csrc_sha": csrc_hash()}
        cur[config] = ent
        json.dump(cur, open(tj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
