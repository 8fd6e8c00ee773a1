#!/usr/bin/env python
"""bench.py -- fp64 HEC SpMV throughput on B200 (BASELINE.json metric:
"fp64 HEC SpMV GFLOP/s and HBM GB/s (% of roofline) at 1/2/4/8 B200").

A step = one y = A x over the whole workload (SURVEY.md §8(a) rows a6-a7 at
N = 1; a6-a10 at N > 1: halo export + exchange -- the peer-memory push kernel,
or pack + NCCL with --transport nccl -- interior and boundary SpMV).
Setup rows a1-a5 (validation, partition, plan, conversion, upload) run once
before timing, as the paper's SpMV timings exclude them.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config poisson3d_256]
  python bench.py --impl reference ...   # the CPU oracle on the same workload

Prints ONE JSON line (rank 0).  N > 1 is launched by torchrun (one process per
GPU; NCCL process group); the row partition is z-slabs (GRID) for grids,
CONTIG_NNZ otherwise.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import hecgen  # noqa: E402

METRIC = "fp64 HEC SpMV GFLOP/s and HBM GB/s (% of roofline) at 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="hec", choices=["hec", "reference"])
    ap.add_argument("--config", default="poisson3d_256", choices=sorted(hecgen.CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks/e2e/cpu)")
    ap.add_argument("--scramble", type=int, default=None,
                    help="apply a seeded random symmetric permutation to the workload (NEXT-4 experiment)")
    ap.add_argument("--reorder", choices=["rcm"], default=None,
                    help="reorder the workload with reverse Cuthill-McKee before converting (NEXT-4)")
    ap.add_argument("--formats", default=None,
                    help="'all' or comma-separated configs: per-format SpMV table (NEXT-2, Table 3 analog)")
    ap.add_argument("--solver", choices=["cg", "bicgstab"], default=None,
                    help="measure Krylov iterations/s instead of the SpMV (NEXT-1)")
    ap.add_argument("--jacobi", type=float, default=None, metavar="OMEGA",
                    help="NEXT-3: time damped-Jacobi sweeps (hec_jacobi) with this omega")
    ap.add_argument("--ell-width", type=int, default=None,
                    help="experiment: FIXED ELL width instead of the BG3 rule (reading A1)")
    ap.add_argument("--transport", choices=["p2p", "nccl", "both"], default="p2p",
                    help="N > 1 halo exchange: peer-memory push kernel over NVLink (default), NCCL send/recv, "
                         "or both timed in one run (NCCL first, then the same handle switched to p2p)")
    ap.add_argument("--no-ncu", action="store_true",
                    help="skip the in-run ncu pass that measures roofline.traffic (dram bytes per launch)")
    ap.add_argument("--no-anchor", action="store_true",
                    help="skip the paper-anchor leg (150^3 GPU / serial speedup beside Table 3's 13.63x)")
    ap.add_argument("--partition", choices=["auto", "nnz", "cost"], default="auto",
                    help="N > 1, non-grid matrices: CONTIG_NNZ (auto, reading A9) or CONTIG_COST (DESIGN §6)")
    ap.add_argument("--dist", action="store_true",
                    help="use the distributed path (hec_spmv_dist under torchrun) even with one GPU")
    return ap.parse_args()


def workload_config(name, A, x_h, world: int = 1):
    """The line's `config`: the workload's identity only (same keys and values
    on the product arm and the reference arm), with the FNV-1a checksums of
    the CSR arrays and x, and the GPU arm's L2 policy (flush iff a rank's
    inputs are < 4x L2).  Run details go under the line's `run` key."""
    alg = algorithmic_bytes(A.nnz, A.n_rows, A.n_cols) // max(1, world)
    l2 = (f"inputs {alg / 1e9:.2f} GB per GPU > 4x the {L2_BYTES / 2**20:.0f} MiB L2: no flush between steps"
          if alg >= 4 * L2_BYTES else
          f"inputs {alg / 1e9:.3f} GB per GPU < 4x L2: GPU arm flushes L2 ({4 * L2_BYTES / 2**20:.0f} MiB write + read) "
          f"before every step, outside the timed pair")
    return {"workload": name, "n_rows": A.n_rows, "n_cols": A.n_cols, "nnz": A.nnz, "l2": l2,
            "checksum": A.checksum(), "x_checksum": hecgen.fnv1a(x_h)}


def grid_of(A):
    return A.grid if A.grid is not None else None


def algorithmic_bytes(nnz, n_rows, n_cols):
    """values + indices + x read once + y written once."""
    return 12 * nnz + 8 * n_cols + 8 * n_rows


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def csrc_hash() -> str:
    """sha256[:16] over the product's native sources (csrc/ + include/): keys the
    committed ncu traffic so a stale capture is never reported for new code."""
    import glob
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_1606_00545_b200", "csrc", "*")) +
                   glob.glob(os.path.join(ROOT, "include", "*.h")))
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def ncu_traffic_committed(config: str):
    """Fallback: dram__bytes_read.sum + dram__bytes_write.sum per step from the
    committed ncu captures (profiles/ncu_traffic.json), used ONLY when the
    capture's csrc_sha matches the current native sources."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p)).get(config, {})
    except Exception:
        return None, None, "no committed capture"
    if d.get("csrc_sha") != csrc_hash():
        return None, None, f"committed capture is for csrc {d.get('csrc_sha')}, not {csrc_hash()} (stale: dropped)"
    return (d.get("dram_bytes_per_step"), {k: v["dram_bytes_per_launch"] for k, v in d.get("kernels", {}).items()},
            f"profiles/ncu_traffic.json (csrc {d.get('csrc_sha')})")


def ncu_traffic_live(config: str, launches_per_step: int, timeout_s: float = 300.0):
    """In-run measurement of roofline.traffic: re-runs this bench (--profile, 2
    warm-up + 3 timed steps) under `ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum,gpu__time_duration.sum` restricted to the HEC
    kernels, and takes the LAST step's launches (warm caches, the timed
    configuration).  Returns (bytes per step, {kernel: bytes}, {kernel: ncu
    ms}, source) or Nones with the reason."""
    import csv
    import shutil
    import tempfile
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if ncu is None:
        return None, None, None, "ncu not found"
    log = tempfile.NamedTemporaryFile(prefix="hec_ncu_", suffix=".csv", delete=False).name
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--csv", "--log-file", log, "--kernel-name-base", "demangled",
           "-k", "regex:hec::", sys.executable, os.path.abspath(__file__), "--profile", "--config", config,
           "--steps", "3", "--warmup", "2"]
    try:
        r = subprocess.run(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.PIPE, timeout=timeout_s, text=True)
        rows = list(csv.reader(l for l in open(log) if l.startswith('"')))
    except Exception as e:
        return None, None, None, f"ncu pass failed: {str(e)[:120]}"
    finally:
        try:
            os.unlink(log)
        except OSError:
            pass
    if not rows or r.returncode != 0:
        return None, None, None, f"ncu pass rc={r.returncode}: {r.stderr[-160:] if r.stderr else ''}"
    hdr = rows[0]
    iid, ik, im, iv = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    for row in rows[1:]:
        k = per.setdefault(int(row[iid]), {"kernel": row[ik]})
        k[row[im]] = float(row[iv].replace(",", ""))
    # every libhec kernel of the child's 5 SpMV steps (2 warm-up + 3): the
    # launches per step are counted, not assumed; the last step's are summed
    counted = len(per) / 5.0
    lps = int(round(counted)) if counted >= 1 else launches_per_step
    ids = sorted(per)[-lps:]
    split, times = {}, {}
    for i in ids:
        k = per[i]
        name = k["kernel"].replace("void ", "").split("<")[0].split("(")[0].replace("hec::", "").strip()
        split[name] = split.get(name, 0) + int(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0))
        times[name] = round(times.get(name, 0.0) + k.get("gpu__time_duration.sum", 0.0) * 1e-6, 5)  # ns -> ms
    times["launches_per_step_counted"] = counted
    return (sum(split.values()), split, times,
            f"measured in this run: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over every libhec "
            f"kernel (hec::*) of 5 steps: {counted:g} launch(es)/step counted; the last step's summed")


class L2Flusher:
    """Between timed steps: write a 4x-L2 buffer (evicts everything), then read
    another one so the dirty lines are written back before the next timed
    step instead of inside it."""

    def __init__(self, device):
        import torch
        self.w = torch.empty(4 * L2_BYTES // 8, dtype=torch.float64, device=device)
        self.r = torch.zeros(4 * L2_BYTES // 8, dtype=torch.float64, device=device)

    def __call__(self):
        self.w.zero_()
        self.r.sum()


# -------------------------------------------------------------- clocks ----
class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------- cpu baseline ----
def host_description() -> dict:
    """lscpu model name, sockets, cores, threads and NUMA nodes
    of the host the CPU legs run on (read at run time)."""
    info = {"logical_cpus": os.cpu_count(), "usable_cpus": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        keys = {"Model name": "model", "Socket(s)": "sockets", "Core(s) per socket": "cores_per_socket",
                "Thread(s) per core": "threads_per_core", "NUMA node(s)": "numa_nodes", "CPU max MHz": "max_mhz"}
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in keys and keys[k.strip()] not in info:
                info[keys[k.strip()]] = v.strip()
    except Exception as e:
        info["lscpu_error"] = str(e)[:80]
    return info


class pinned_core:
    """`taskset -c <core>` for the calling thread (Linux sched_setaffinity on
    pid 0 applies to the calling thread), restored on exit: the serial oracle
    leg runs on one pinned core (the paper's "CPU sequential
    running time")."""

    def __init__(self):
        self.prev = os.sched_getaffinity(0)
        self.core = min(self.prev)

    def __enter__(self):
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.prev)


def serial_oracle_ms(A, x, budget_s: float, max_s: float = 30.0):
    """The oracle O1 as it stands (serial C), whole matrix, on one pinned core:
    1 warm-up, then repetitions until ~budget_s; (best ms, mean ms, reps, core)."""
    import oracle
    oracle._load()                       # libgomp sizes its pool from the UNPINNED mask
    with pinned_core() as pc:
        oracle.csr_spmv(A, x)            # warm-up
        times = []
        t_all = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            oracle.csr_spmv(A, x)
            times.append(time.perf_counter() - t0)
            el = time.perf_counter() - t_all
            if (el >= budget_s and len(times) >= 3) or el + times[-1] > max_s:
                break
    return min(times) * 1e3, sum(times) / len(times) * 1e3, len(times), pc.core


def cpu_oracle_rate(A, x, budget_s=12.0, max_s=30.0):
    """(i) the oracle O1 as it stands, serial, pinned to one core, on the whole
    matrix repeated for ~budget_s; (ii) the same O1 rows over all host threads
    (OpenMP, bit-identical), ~3 s.  Plus the lscpu record."""
    import oracle
    best, mean, reps, core = serial_oracle_ms(A, x, budget_s, max_s)
    par_times, threads = [], 1
    t_all = time.perf_counter()
    while time.perf_counter() - t_all < 3.0 and len(par_times) < 50:
        t0 = time.perf_counter()
        _, threads = oracle.csr_spmv_parallel(A, x)
        par_times.append(time.perf_counter() - t0)
    pbest = min(par_times)
    alg = algorithmic_bytes(A.nnz, A.n_rows, A.n_cols)
    return {"value": round(2 * A.nnz / (best * 1e-3) / 1e9, 4), "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
            "sample": f"whole {A.name} matrix ({A.n_rows} rows, {A.nnz} nnz), serial O1 pinned to core {core} "
                      f"(taskset equivalent), 1 warm-up + {reps} reps, best {best:.1f} ms, mean {mean:.1f} ms",
            "gbs": round(alg / (best * 1e-3) / 1e9, 2),
            "mean_gflops": round(2 * A.nnz / (mean * 1e-3) / 1e9, 4),
            "host": host_description(),
            "parallel": {"value": round(2 * A.nnz / pbest / 1e9, 4), "unit": "GFLOP/s", "cores": threads,
                         "kind": "oracle O1 rows over OpenMP threads (bit-identical)",
                         "sample": f"{len(par_times)} reps, best {pbest * 1e3:.1f} ms"}}


def paper_anchor(dev: int, budget_s: float = 4.0):
    """SURVEY §8(d) paper anchor (context, not a target): the paper's own
    3D_Poisson 150^3 -- GPU hec_spmv time (cold L2, median of 30) and
    the serial oracle on one pinned core -- and their ratio in the paper's
    speedup definition (CPU sequential time / GPU time), beside Table 3's
    HEC value for 3D_Poisson, 13.63x (Tesla C2050/C2070 vs a Xeon X5570
    core) and "most ... over 10 and the highest ... 18"."""
    import torch
    import paper_1606_00545_b200 as hec
    A = hecgen.poisson3d(150, 150, 150)
    x_h = hecgen.vector(A.n_cols, "uniform", seed=1606)
    M = hec.from_csr(A, device=dev)
    x = torch.from_numpy(x_h).to(f"cuda:{dev}")
    y = torch.empty(A.n_rows, dtype=torch.float64, device=f"cuda:{dev}")
    fl = L2Flusher(f"cuda:{dev}")
    for _ in range(5):
        M.spmv(x, y)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
    for a, b in ev:
        fl()
        a.record()
        M.spmv(x, y)
        b.record()
    torch.cuda.synchronize()
    gpu_ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    best, mean, reps, core = serial_oracle_ms(A, x_h, budget_s)
    M.free()
    return {"config": "poisson3d_150 (the paper's 3D_Poisson, P:406)", "gpu_ms": round(gpu_ms, 5),
            "gpu_l2": "cold (flushed), median of 30", "serial_oracle_ms": round(best, 3),
            "serial_sample": f"O1 pinned to core {core}, best of {reps}",
            "speedup_vs_serial": round(best / gpu_ms, 1),
            "paper_speedup_hec_3d_poisson": 13.63, "paper_claim": "most HEC speedups over 10, highest 18 (P:413)",
            "paper_hardware": "NVIDIA Tesla C2050/C2070 vs Intel Xeon X5570 serial -O3 (P:378-382)",
            "note": "context only: different hardware; the CPU side here is the oracle as it stands"}


# ------------------------------------------------------------ reference ----
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    A = hecgen.CONFIGS[args.config]()
    x = hecgen.vector(A.n_cols, "uniform", seed=1606)
    oracle.csr_spmv(A, x, 0, min(1024, A.n_rows))
    # calibrate the serial rate, then size each step so the run stays ~<= 90 s
    t0 = time.perf_counter()
    r1 = min(A.n_rows, 1 << 20)
    oracle.csr_spmv(A, x, 0, r1)
    dt = max(time.perf_counter() - t0, 1e-6)
    nnz_rate = A.row_ptr[r1] / dt
    budget = 90.0 / max(1, args.steps + args.warmup)
    rows = A.n_rows
    if A.nnz / nnz_rate > budget:
        rows = int(np.searchsorted(A.row_ptr, nnz_rate * budget))
        rows = max(1, min(A.n_rows, rows))
    starts = np.linspace(0, A.n_rows - rows, num=max(1, args.steps + args.warmup)).astype(np.int64)
    for k in range(args.warmup):
        r0 = int(starts[k])
        oracle.csr_spmv(A, x, r0, r0 + rows)
    flops, total = 0, 0.0
    with pinned_core() as pc:
        for k in range(args.warmup, args.warmup + args.steps):
            r0 = int(starts[k])
            t0 = time.perf_counter()
            oracle.csr_spmv(A, x, r0, r0 + rows)
            total += time.perf_counter() - t0
            flops += 2 * int(A.row_ptr[r0 + rows] - A.row_ptr[r0])
    value = flops / total / 1e9
    sample = (f"{rows} contiguous rows of {A.name} per step ({'whole matrix' if rows == A.n_rows else 'bounded sample'}), "
              f"serial O1 (spmv_oracle.c, -O2 -ffp-contract=off), pinned to core {pc.core}")
    line = {"metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": workload_config(args.config, A, x, max(1, args.gpus)),
            "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                             "sample": sample, "host": host_description()},
            "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ single GPU ----
def run_single(args):
    import torch
    import paper_1606_00545_b200 as hec
    dev = 0
    torch.cuda.set_device(dev)
    t_setup = time.perf_counter()
    A = hecgen.CONFIGS[args.config]()
    reorder_info = None
    if args.scramble is not None or args.reorder:
        # NEXT-4 experiment: a random symmetric permutation of the workload
        # (input generation), then optionally the RCM reordering (setup)
        def halo8(M):
            P = hec.partition(M, 8, hec.PART_CONTIG_NNZ)
            return int(sum(P.part_info(p).n_halo for p in range(8)))
        reorder_info = {}
        if args.scramble is not None:
            perm = np.random.default_rng(args.scramble).permutation(A.n_rows).astype(np.int32)
            A = hec.permute(A, perm)
            A.name = f"{args.config}_scrambled{args.scramble}"
            reorder_info["scrambled_seed"] = args.scramble
        reorder_info["halo_entries_p8_before"] = halo8(A)
        if args.reorder == "rcm":
            t0 = time.perf_counter()
            A = hec.permute(A, hec.reorder_rcm(A))
            reorder_info["rcm_s"] = round(time.perf_counter() - t0, 2)
            reorder_info["halo_entries_p8_after"] = halo8(A)
        A.name = A.name or args.config
    t_gen = time.perf_counter() - t_setup
    x_h = hecgen.vector(A.n_cols, "uniform", seed=1606)
    stream = torch.cuda.Stream()
    t0 = time.perf_counter()
    o = hec.opts(hec.WIDTH_FIXED, 20, args.ell_width) if args.ell_width is not None else None
    M = hec.from_csr(A, o, device=dev, stream=stream)
    t_conv = time.perf_counter() - t0
    x = torch.from_numpy(x_h).to(f"cuda:{dev}")
    y = torch.empty(A.n_rows, dtype=torch.float64, device=f"cuda:{dev}")
    torch.cuda.synchronize()
    launches_per_step = M.launches
    alg = algorithmic_bytes(A.nnz, A.n_rows, A.n_cols)
    inf = M.info
    fmt_bytes = 12 * inf.ell_width * inf.ell_stride + 12 * inf.tail_nnz + 8 * (inf.tail_rows + 1) \
        + 4 * inf.tail_rows + 8 * A.n_cols + 8 * A.n_rows + 16 * inf.tail_rows

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            M.spmv(x, y, stream)
    torch.cuda.synchronize()

    K = args.steps
    # L2 policy: inputs far larger than L2 need no flush; otherwise write a
    # 4x-L2 scratch buffer before every step, outside that step's event pair
    flush = alg < 4 * L2_BYTES
    flusher = L2Flusher(f"cuda:{dev}") if flush else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    sampler = ClockSampler(dev) if not args.profile else None
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
        time.sleep(0.02)
    with torch.cuda.stream(stream):
        for k in range(K):
            if flush:
                flusher()
            ev[k][0].record(stream)
            M.spmv(x, y, stream)
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    per = [a.elapsed_time(b) for a, b in ev]  # ms, one step each
    ms_step = sum(per) / K
    gflops = 2 * A.nnz / (ms_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    # dominant kernel: the ELL kernel (the only launch per step when there is no tail)
    mean_launch_ms = statistics.mean(per)
    achieved = alg / (mean_launch_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": None, "traffic_by_kernel": None,
            "kernel": "ell_kernel" + ("" if launches_per_step == 1 else "+tail_kernel (step)"),
            "algorithmic_bytes_per_launch": alg, "format_bytes_per_launch": fmt_bytes,
            "peak_source": peak_src, "frac_of_8TBs_nominal": round(achieved / 8000.0, 4),
            "median_step_ms": round(statistics.median(per), 5),
            "p10_step_ms": round(float(np.percentile(per, 10)), 5),
            "p90_step_ms": round(float(np.percentile(per, 90)), 5)}

    # SURVEY §8(d) secondary: warm timing, back-to-back SpMVs replayed from one
    # captured CUDA graph (no flush), reported beside the primary number
    if not args.profile:
        try:
            G = 50
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(G):
                    M.spmv(x, y, stream)
            g.replay()
            torch.cuda.synchronize()
            w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                w0.record(stream)
                for _ in range(4):
                    g.replay()
                w1.record(stream)
            torch.cuda.synchronize()
            roof["warm_graph_ms_per_spmv"] = round(w0.elapsed_time(w1) / (4 * G), 5)
            del g
        except Exception as e:  # capture is diagnostic only
            roof["warm_graph_ms_per_spmv"] = None
            roof["warm_graph_error"] = str(e)[:200]

    # end to end through the public API with HOST buffers (pinned), copies inside
    e2e = None
    if not args.no_e2e and not args.profile:
        xp = torch.from_numpy(x_h).pin_memory()
        yp = torch.empty(A.n_rows, dtype=torch.float64).pin_memory()
        for _ in range(min(3, args.warmup)):
            M.spmv_host(xp, yp, stream)
        Ke = max(3, min(K, 50))
        t0 = time.perf_counter()
        for _ in range(Ke):
            M.spmv_host(xp, yp, stream)
        dt = (time.perf_counter() - t0) / Ke
        e2e = {"value": round(2 * A.nnz / dt / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": 8 * A.n_cols, "d2h_bytes_per_step": 8 * A.n_rows,
               "ms_per_step": round(dt * 1e3, 4), "steps": Ke, "api": "hec_spmv_host (pinned host x, y)"}

    # roofline.traffic: dram bytes per launch measured by an ncu pass of this
    # same bench (subprocess), else the committed capture if it is for these
    # exact native sources, else null
    if not args.profile:
        if args.no_ncu or args.scramble is not None or args.reorder or args.ell_width is not None:
            tr, split, ncu_ms, src = None, None, None, "skipped (--no-ncu or a non-default workload)"
        else:
            M.free()  # release the device copy while the ncu child builds its own
            torch.cuda.empty_cache()
            tr, split, ncu_ms, src = ncu_traffic_live(args.config, launches_per_step)
            if tr is None:
                reason = src
                tr, split, src = ncu_traffic_committed(args.config)
                src = f"{src} (live pass unavailable: {reason})"
                ncu_ms = None
        if ncu_ms and "launches_per_step_counted" in ncu_ms:
            counted = ncu_ms.pop("launches_per_step_counted")
            roof["gpu_launches_evidence"] = {"ncu_launches_per_step": counted, "claimed_per_step": launches_per_step,
                                             "agrees": abs(counted - launches_per_step) < 1e-9}
        roof.update({"traffic": tr, "traffic_by_kernel": split, "traffic_source": src,
                     "ncu_ms_by_kernel": ncu_ms, "csrc_sha": csrc_hash()})
        if tr:
            roof["traffic_over_algorithmic"] = round(tr / alg, 4)

    cpu = None
    if not args.no_cpu_baseline and not args.profile:
        cpu = cpu_oracle_rate(A, x_h)
        cpu["gpu_speedup_vs_serial"] = round(2 * A.nnz / (ms_step * 1e-3) / 1e9 / cpu["value"], 1)
    anchor = None
    if not args.no_anchor and not args.profile:
        anchor = paper_anchor(dev)

    line = {"metric": METRIC, "value": round(gflops, 2), "unit": "GFLOP/s", "n_gpus": 1, "steps": K,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, A, x_h),
            "run": {"parallelism": "1 GPU", "ell_width": inf.ell_width, "ell_stride": inf.ell_stride,
                    "tail_rows": inf.tail_rows, "tail_nnz": inf.tail_nnz,
                    "width_policy": "BG3 (A1)" if args.ell_width is None else f"FIXED {args.ell_width} (experiment)",
                    "setup_s": {"generate": round(t_gen, 2), "convert_upload": round(t_conv, 2)},
                    "reorder": reorder_info},
            "gbs": round(alg / (ms_step * 1e-3) / 1e9, 1),
            "roofline": roof, "gpu_launches": K * launches_per_step,
            "e2e": e2e, "cpu_baseline": cpu, "paper_anchor": anchor,
            "clocks": sampler.summary() if sampler else None}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- multi GPU ----
def time_dist_steps(D, x, y, stream, K, flusher, dist, torch):
    """SURVEY §8(d) multi-GPU protocol, per repetition: every rank scrubs L2
    (when its working set is < 4x L2), a tiny NCCL all-reduce aligns the ranks
    on the device, then each rank times ONE hec_spmv_dist with CUDA events on
    the launch stream.  T(P) of a repetition = the max over ranks (all-reduce
    MAX of the per-repetition times).  Returns the per-repetition maxima (ms)
    and the wall time between the bracketing barriers (s)."""
    align = torch.zeros(1, dtype=torch.float32, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(stream):
        for k in range(K):
            if flusher:
                flusher()  # outside the timed pair: evicts this rank's matrix from L2
            dist.all_reduce(align)  # the stream waits until every rank got here
            ev[k][0].record(stream)
            D.spmv(x, y, stream)
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    wall = time.perf_counter() - t0
    per = torch.tensor([a.elapsed_time(b) for a, b in ev], dtype=torch.float64, device="cuda")
    dist.all_reduce(per, op=dist.ReduceOp.MAX)
    return per.cpu().numpy(), wall


def dist_overlap(D, x, y, stream, flusher, dist, torch, reps=10):
    """The a10 overlap evidence: hec_dist_set_timing's events on each rank
    (interior rows end / exchange + boundary rows end, both from the call's
    start), median of `reps` aligned calls; per rank, then the max over ranks
    of the exposed exchange time max(0, comm - interior)."""
    D.set_timing(True)
    align = torch.zeros(1, dtype=torch.float32, device="cuda")
    it, co = [], []
    for _ in range(reps):
        with torch.cuda.stream(stream):
            if flusher:
                flusher()
            dist.all_reduce(align)
            D.spmv(x, y, stream)
        a, b = D.phase_times()
        it.append(a)
        co.append(b)
    D.set_timing(False)
    mine = torch.tensor([statistics.median(it), statistics.median(co)], dtype=torch.float64, device="cuda")
    allr = [torch.zeros_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(allr, mine)
    per = [(round(float(t[0]), 5), round(float(t[1]), 5)) for t in allr]
    exposed = [max(0.0, c - i) for i, c in per if c >= 0]
    return {"what": "per rank: ms from the call's start to the end of the interior rows / of exchange + boundary "
                    "rows (CUDA events on the two streams, hec_dist_phase_times), median of 10 aligned calls",
            "interior_ms": [p[0] for p in per], "exchange_boundary_ms": [p[1] for p in per],
            "exposed_ms_max": round(max(exposed), 5) if exposed else None}


def dist_parity(A, x_h, y, r0, r1, dist, torch):
    """Every row of every rank against the serial C oracle O1 (tolerance
    1e-12 (|A||x|)_i): each rank checks its own rows [r0, r1); the bad-row
    counts are summed over ranks.  Makes the first N > 1 run self-proving."""
    import oracle
    got = y.cpu().numpy()
    ref = oracle.csr_spmv(A, x_h, r0, r1)
    tol = oracle.tolerance(A, x_h, r0, r1)
    bad = torch.tensor([float(np.count_nonzero(~(np.abs(got - ref) <= tol))), float(r1 - r0)],
                       dtype=torch.float64, device="cuda")
    dist.all_reduce(bad)
    return {"rows_checked": int(bad[1].item()), "bad_rows": int(bad[0].item()),
            "vs": "oracle O1 (serial C), every row, |y - y_ref| <= 1e-12 (|A||x|)_i", "ok": bad[0].item() == 0}


def run_multi(args):
    import torch
    import torch.distributed as dist
    import paper_1606_00545_b200 as hec
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    A = hecgen.CONFIGS[args.config]()
    kind = (hec.PART_GRID if A.grid is not None else
            hec.PART_CONTIG_COST if args.partition == "cost" else hec.PART_CONTIG_NNZ)
    plan = hec.partition(A, world, kind, A.grid)
    obj = [hec.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    D = hec.Dist(A, plan, rank, obj[0], local)
    comm_ranks, nccl_version = D.comm_size()
    x_h = hecgen.vector(A.n_cols, "uniform", seed=1606)
    r0, r1 = D.info.r0, D.info.r1
    x = torch.from_numpy(x_h[r0:r1].copy()).cuda()
    y = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
    stream = torch.cuda.Stream()
    # L2 policy: flush between steps unless this rank's working set is far larger than L2
    flush = D.info.algorithmic_bytes < 4 * L2_BYTES
    flusher = L2Flusher("cuda") if flush else None
    K = args.steps
    # transports to time: NCCL send/recv (the handle as created), then the
    # peer-memory push (the same handle switched by hec_dist_enable_p2p)
    order = {"p2p": ["p2p"], "nccl": ["nccl"], "both": ["nccl", "p2p"]}[args.transport] if world > 1 else ["none"]
    results, sampler = {}, None
    for t in order:
        if t == "p2p":
            ok = 1.0
            try:
                D.enable_p2p()
            except hec.HecError as e:
                print(f"rank {rank}: peer-memory transport unavailable ({e})", file=sys.stderr)
                ok = 0.0
            okt = torch.tensor([ok], device="cuda")
            dist.all_reduce(okt, op=dist.ReduceOp.MIN)
            if okt.item() < 0.5:
                results[t] = {"unavailable": "hec_dist_enable_p2p failed on some rank (see stderr)"}
                if len(order) == 1:  # fall back to the NCCL transport on a fresh handle
                    D.free()
                    obj = [hec.nccl_unique_id() if rank == 0 else None]
                    dist.broadcast_object_list(obj, src=0)
                    D = hec.Dist(A, plan, rank, obj[0], local)
                    t = "nccl"
                else:
                    continue
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                D.spmv(x, y, stream)
        torch.cuda.synchronize()
        sampler = ClockSampler(local) if not args.profile else None
        if sampler:
            sampler.__enter__()
        per, wall = time_dist_steps(D, x, y, stream, K, flusher, dist, torch)
        if sampler:
            sampler.__exit__()
        D.check()  # raises if a peer-memory halo wait timed out (the results would be garbage)
        par = dist_parity(A, x_h, y, r0, r1, dist, torch)
        overlap = dist_overlap(D, x, y, stream, flusher, dist, torch) if world > 1 else None
        ms_mean = float(np.mean(per))
        results[t] = {"ms_per_step": round(ms_mean, 5), "median_ms": round(float(np.median(per)), 5),
                      "p10_ms": round(float(np.percentile(per, 10)), 5),
                      "p90_ms": round(float(np.percentile(per, 90)), 5),
                      "gflops": round(2 * A.nnz / (ms_mean * 1e-3) / 1e9, 2),
                      "wall_s_between_barriers": round(wall, 4), "parity": par, "overlap": overlap,
                      "launches_per_step": D.info.launches, "clocks": sampler.summary() if sampler else None}
    head = "p2p" if "p2p" in results and "ms_per_step" in results["p2p"] else \
        ("nccl" if "nccl" in results else order[-1])
    hr = results[head]
    alg_loc = torch.tensor([float(D.info.algorithmic_bytes)], dtype=torch.float64, device="cuda")
    dist.all_reduce(alg_loc)
    # end to end through the public C ABI with HOST buffers: hec_spmv_dist_host
    # (H2D of this rank's x slice, the distributed product, D2H of its y slice)
    e2e = None
    if not args.no_e2e and not args.profile:
        xp = torch.from_numpy(x_h[r0:r1].copy()).pin_memory()
        yp = torch.empty(r1 - r0, dtype=torch.float64).pin_memory()
        Ke = max(3, min(K, 50))
        for _ in range(2):
            D.spmv_host(xp, yp, stream)
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(Ke):
            D.spmv_host(xp, yp, stream)
        dt = torch.tensor([(time.perf_counter() - t0) / Ke], dtype=torch.float64, device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": round(2 * A.nnz / float(dt.item()) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": 8 * A.n_cols, "d2h_bytes_per_step": 8 * A.n_rows,
               "ms_per_step": round(float(dt.item()) * 1e3, 4), "steps": Ke,
               "api": "hec_spmv_dist_host (pinned host slices; H2D + product + D2H per step), max over ranks"}
    if rank == 0:
        ms_step = hr["ms_per_step"]
        gflops = 2 * A.nnz / (ms_step * 1e-3) / 1e9
        peak, peak_src = measured_peak()
        achieved = float(alg_loc.item()) / world / (ms_step * 1e-3) / 1e9
        pname = 'GRID slabs' if kind == hec.PART_GRID else 'CONTIG_COST' if kind == hec.PART_CONTIG_COST else 'CONTIG_NNZ'
        line = {"metric": METRIC, "value": round(gflops, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": K,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(args.config, A, x_h, world),
                "run": {"parallelism": f"row partition x{world} ({pname}), "
                                          + {"p2p": "peer-memory halo push over NVLink",
                                             "nccl": "NCCL send/recv halo exchange",
                                             "none": "single rank (no exchange)"}[head],
                           "transport": head,
                           "timing": "per repetition: L2 scrub (if needed), NCCL all-reduce alignment, event pair "
                                     "around one hec_spmv_dist; T = max over ranks per repetition; value from the mean",
                           "l2": ("L2 flushed (504 MiB write + 504 MiB read) before every step, outside the timed pair" if flush
                                  else "per-rank inputs > 4x L2, no flush")},
                "gbs": round(float(alg_loc.item()) / (ms_step * 1e-3) / 1e9, 1),
                "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                             "frac": round(achieved / peak, 4), "traffic": None,
                             "kernel": "whole step per rank (interior + boundary SpMV, halo exchange)",
                             "peak_source": peak_src, "median_step_ms": hr["median_ms"]},
                "parity": hr["parity"], "transports": results,
                "nccl": {"version": nccl_version, "comm_ranks": comm_ranks},
                "gpu_launches": K * hr["launches_per_step"], "e2e": e2e, "cpu_baseline": None,
                "clocks": hr["clocks"]}
        print(json.dumps(line), flush=True)
    D.free()
    dist.barrier()
    dist.destroy_process_group()
    return 0 if all(r.get("parity", {}).get("ok", True) for r in results.values()) else 3


def run_solver(args):
    """NEXT-1 measurement (not the headline): a fixed number of Krylov
    iterations (BiCGSTAB = Alg. 4 with M = I, or CG) on the workload, one GPU.
    Reports iterations/s and the bytes the iteration must move (SpMVs +
    vector passes) against the HBM peak; the oracle's serial iteration rate on
    the same matrix (bounded: a few iterations) beside it."""
    import torch
    import paper_1606_00545_b200 as hec
    torch.cuda.set_device(0)
    A = hecgen.CONFIGS[args.config]()
    b_h = hecgen.vector(A.n_rows, "uniform", seed=7)
    M = hec.from_csr(A)
    b = torch.from_numpy(b_h).cuda()
    x = torch.zeros(A.n_rows, dtype=torch.float64, device="cuda")
    solve = M.cg if args.solver == "cg" else M.bicgstab
    solve(b, x, 0.0, max(1, args.warmup))                      # warm-up iterations
    torch.cuda.synchronize()
    K = args.steps
    x.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record()
        info = solve(b, x, 0.0, K)                               # tol 0: exactly K iterations
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    n, alg = A.n_rows, algorithmic_bytes(A.nnz, A.n_rows, A.n_cols)
    # per iteration: CG = 1 SpMV + dot(p,q) 2n + x,r update 6n + p update 3n (doubles)
    #                BiCGSTAB = 2 SpMV + p 4n + dot 2n + s 3n + 2 dots 3n + x,r 7n
    per_it = alg + 8 * n * 11 if args.solver == "cg" else 2 * alg + 8 * n * 19
    it_s = info.iterations / (ms * 1e-3)
    peak, peak_src = measured_peak()
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import krylov_ref as KR
        t0 = time.perf_counter()
        its = 2
        (KR.cg if args.solver == "cg" else KR.bicgstab)(A, b_h, np.zeros(n), 0.0, its)
        dt = time.perf_counter() - t0
        cpu = {"value": round(its / dt, 4), "unit": "iterations/s", "cores": 1, "kind": "oracle",
               "sample": f"{its} iterations of oracle/krylov_ref.{args.solver} on {A.name} (serial O1 SpMV, "
                         f"plain-Python dots), {dt:.1f} s"}
    line = {"metric": f"fp64 {args.solver} iterations/s (HEC SpMV consumer, NEXT-1)", "value": round(it_s, 2),
            "unit": "iterations/s", "n_gpus": 1, "steps": info.iterations, "warmup": args.warmup,
            "ms_per_step": round(ms / max(1, info.iterations), 5), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n_rows": n, "nnz": A.nnz, "solver": args.solver,
                       "tol": 0.0, "rel_residual_at_end": info.rel_residual},
            "roofline": {"bound": "hbm", "achieved": round(per_it * it_s / 1e9, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(per_it * it_s / 1e9 / peak, 4), "traffic": None,
                         "kernel": "whole iteration (SpMV + fused vector passes)",
                         "algorithmic_bytes_per_iteration": per_it, "peak_source": peak_src},
            "cpu_baseline": cpu,
            # per iteration: CG = SpMV + 3 fused passes; BiCGSTAB = 2 SpMV + 6 passes + 1 step kernel
            "gpu_launches": info.iterations * (M.launches + 3 if args.solver == "cg" else 2 * M.launches + 7),
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


def run_jacobi(args):
    """NEXT-3 measurement (not the headline): damped-Jacobi sweeps x <- x +
    omega D^-1 (b - A x) (hec_jacobi, the SpMV with its Jacobi epilogue),
    ping-pong over K sweeps, per-sweep event pairs (cold L2 below 4x L2).
    Algorithmic bytes per sweep = the SpMV's (12 nnz + 8 n_cols + 8 n_rows)
    + b and d (16 n).  The plain SpMV on the same matrix is timed beside it."""
    import torch
    from oracle import jacobi_ref as JR
    import paper_1606_00545_b200 as hec
    torch.cuda.set_device(0)
    A = hecgen.CONFIGS[args.config]()
    n = A.n_rows
    M = hec.from_csr(A)
    b_h = hecgen.vector(n, "uniform", seed=7)
    x_h = hecgen.vector(n, "uniform", seed=8)
    b = torch.from_numpy(b_h).cuda()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    M.diag(d)
    u, v = torch.from_numpy(x_h).cuda(), torch.empty(n, dtype=torch.float64, device="cuda")
    alg = algorithmic_bytes(A.nnz, n, A.n_cols) + 16 * n
    cold = alg < 4 * L2_BYTES
    flusher = L2Flusher("cuda:0") if cold else None
    # one checked sweep (sampled rows against the oracle), then warm-up
    M.jacobi(d, b, u, v, args.jacobi)
    r0 = n // 3
    r1 = min(n, r0 + 4000)
    d_s = JR.diag(A, r0, r1)
    ref = JR.jacobi(A, d_s, b_h[r0:r1], x_h, args.jacobi, r0, r1)
    tol = JR.tolerance(A, d_s, b_h[r0:r1], x_h, args.jacobi, r0, r1)
    ok = bool(np.all(np.abs(v.cpu().numpy()[r0:r1] - ref) <= tol))
    for _ in range(max(3, args.warmup)):
        M.jacobi(d, b, u, v, args.jacobi)
        u, v = v, u

    def timed(fn, K):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for e0, e1 in ev:
            if flusher:
                flusher()
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        return sum(e0.elapsed_time(e1) for e0, e1 in ev) / K

    state = [u, v]

    def sweep():
        M.jacobi(d, b, state[0], state[1], args.jacobi)
        state.reverse()
    with ClockSampler(0) as clk:
        ms = timed(sweep, args.steps)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    spmv_ms = timed(lambda: M.spmv(state[0], y), args.steps)
    peak, peak_src = measured_peak()
    gbs = alg / (ms * 1e-3) / 1e9
    line = {"metric": "fp64 damped-Jacobi sweeps/s (HEC SpMV + fused epilogue, NEXT-3)",
            "value": round(1e3 / ms, 2), "unit": "sweeps/s", "n_gpus": 1, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n_rows": n, "nnz": A.nnz, "omega": args.jacobi,
                       "l2": "flushed before every sweep" if cold else "inputs > 4x L2, no flush",
                       "spmv_ms_same_matrix": round(spmv_ms, 5), "parity_sample_ok": ok},
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "traffic": None, "kernel": "ell_kernel<EPI_JACOBI> (+ tail)",
                         "algorithmic_bytes_per_sweep": alg, "peak_source": peak_src},
            "gpu_launches": M.launches * args.steps, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


def run_formats(args):
    """NEXT-2: the paper's Table 3 experiment (SpMV speedup per format)
    on B200 with the synthetic workloads: ELL (w = max row length, no
    remainder), HYB (ELL + COO remainder, Bell & Garland), HEC with the paper's
    literal boundary 20 (CAP policy), and HEC with the default BG3 width.  The
    speedup is the paper's: serial CPU time (the oracle O1, one core) / GPU
    time.  One JSON line per (workload, format); cold L2 below 4x L2."""
    import torch
    import oracle
    import paper_1606_00545_b200 as hec
    torch.cuda.set_device(0)
    configs = args.formats.split(",") if args.formats != "all" else \
        ["poisson2d_64", "spe10", "poisson3d_128", "poisson3d_150", "poisson3d_256", "powerlaw_8M"]
    flusher = L2Flusher("cuda:0")
    free_bytes = torch.cuda.mem_get_info()[0]
    for cfg in configs:
        A = hecgen.CONFIGS[cfg]()
        x_h = hecgen.vector(A.n_cols, "uniform", seed=1606)
        x = torch.from_numpy(x_h).cuda()
        y = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
        alg = algorithmic_bytes(A.nnz, A.n_rows, A.n_cols)
        # serial CPU time of the same product (the paper's speedup denominator)
        reps, t_cpu = 0, 0.0
        while t_cpu < 1.0 and reps < 50:
            t0 = time.perf_counter()
            oracle.csr_spmv(A, x_h)
            t_cpu += time.perf_counter() - t0
            reps += 1
        cpu_ms = t_cpu / reps * 1e3
        max_len = int(np.diff(A.row_ptr).max())
        variants = [("ELL", hec.opts(hec.WIDTH_CAP, max_len), False),
                    ("HYB", hec.opts(), True),
                    ("HEC-20", hec.opts(hec.WIDTH_CAP, 20), False),
                    ("HEC", hec.opts(), False)]
        for name, o, hyb in variants:
            w = min(o.cap, max_len) if o.width_policy == hec.WIDTH_CAP else None
            need = 12 * (w or 0) * A.n_rows
            rec = {"metric": "fp64 SpMV GFLOP/s per format (Table 3 analog)", "workload": cfg, "format": name,
                   "n_rows": A.n_rows, "nnz": A.nnz, "cpu_serial_ms": round(cpu_ms, 3)}
            if need > 0.8 * free_bytes:
                rec["skipped"] = f"ELL width {w} needs {need / 1e9:.0f} GB of slots"
                print(json.dumps(rec), flush=True)
                continue
            M = hec.Matrix(A, o, 0, hyb=hyb)
            cold = alg < 4 * L2_BYTES
            for _ in range(5):
                M.spmv(x, y)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
            for a, b in ev:
                if cold:
                    flusher()
                a.record()
                M.spmv(x, y)
                b.record()
            torch.cuda.synchronize()
            ms = statistics.median(a.elapsed_time(b) for a, b in ev)
            yv = y.cpu().numpy()
            r0 = A.n_rows // 3
            ok = bool(np.all(np.abs(yv[r0:r0 + 2000] - oracle.csr_spmv(A, x_h, r0, min(A.n_rows, r0 + 2000)))
                             <= oracle.tolerance(A, x_h, r0, min(A.n_rows, r0 + 2000))))
            inf = M.info
            rec.update({"gpu_ms": round(ms, 5), "gflops": round(2 * A.nnz / (ms * 1e-3) / 1e9, 2),
                        "alg_gbs": round(alg / (ms * 1e-3) / 1e9, 1), "speedup_vs_serial": round(cpu_ms / ms, 1),
                        "ell_width": inf.ell_width, "tail_rows": inf.tail_rows, "tail_nnz": inf.tail_nnz,
                        "stored_bytes": 12 * inf.ell_width * inf.ell_stride + 12 * inf.tail_nnz +
                        (4 * inf.tail_nnz if hyb else 8 * inf.tail_rows), "l2": "cold" if cold else "inputs > 4x L2",
                        "parity_sample_ok": ok})
            print(json.dumps(rec), flush=True)
            M.free()
        del x, y
        torch.cuda.empty_cache()
    return 0


def main():
    args = parse()
    # stdout carries exactly the JSON line: whatever native code writes to
    # file descriptor 1 (NCCL prints its "NCCL version" banner there) goes to
    # stderr, and Python's stdout keeps the original descriptor
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(json_fd, "w", buffering=1)
    if args.formats:
        return run_formats(args)
    if args.solver:
        return run_solver(args)
    if args.jacobi is not None:
        return run_jacobi(args)
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.dist:
        if "RANK" not in os.environ:
            # self-launch under torchrun
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr=127.0.0.1", "--master-port=29533", __file__] + sys.argv[1:]
            return subprocess.call(cmd, stdout=sys.stdout)
        return run_multi(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
