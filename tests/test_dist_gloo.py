"""Multi-process host logic of the distributed path on CPU (gloo, world_size 2
and 3): every rank builds the product plan independently (it must agree across
ranks), exchanges its halo over the process group with the product's
send/recv lists, and evaluates its interior/boundary sub-HECs (exported from
the product) with the oracle's Alg. 1 evaluation.  The concatenated result
must equal the whole-matrix oracle, bitwise on integer data.
The device kernels of the same path are covered by tests/test_gpu_*.py."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def exchange_halo_host(plan, rank, x_local, group=None):
    """Host-side halo exchange over a torch.distributed process group (gloo),
    following the product plan's send/recv lists -- the same pattern
    hec_spmv_dist runs on the device.  Test infrastructure: returns
    x_halo ordered as recv_cols."""
    import torch
    import torch.distributed as dist
    a = plan.export(rank)
    P = plan.n_parts
    halo = np.empty(len(a.recv_cols), np.float64)
    reqs, bufs, recvs = [], [], []
    for q in range(P):
        lo, hi = int(a.send_off[q]), int(a.send_off[q + 1])
        if hi > lo:
            t = torch.from_numpy(np.ascontiguousarray(x_local[a.send_idx[lo:hi]]))
            bufs.append(t)
            reqs.append(dist.isend(t, dst=q, group=group))
    for q in range(P):
        lo, hi = int(a.recv_off[q]), int(a.recv_off[q + 1])
        if hi > lo:
            t = torch.empty(hi - lo, dtype=torch.float64)
            recvs.append((lo, hi, t))
            reqs.append(dist.irecv(t, src=q, group=group))
    for r in reqs:
        r.wait()
    for lo, hi, t in recvs:
        halo[lo:hi] = t.numpy()
    return halo


def _make(case):
    import hecgen
    if case == "poisson":
        return hecgen.poisson3d(6, 5, 8), (6, 5, 8)
    if case == "powerlaw_int":
        return hecgen.powerlaw(400, integer_values=True, seed=3), None
    return hecgen.spe10(10, 12, 6, seed=2), None


def _worker(rank, world, port, case, out_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import hecgen
        import oracle
        from oracle import hec_ref as H
        import paper_1606_00545_b200 as hec
        A, grid = _make(case)
        kind = hec.PART_GRID if grid else hec.PART_CONTIG_NNZ
        plan = hec.partition(A, world, kind, grid)
        pp = plan.part_ptr()
        # all ranks must hold the same plan
        gathered = [None] * world
        dist.all_gather_object(gathered, pp.tolist())
        assert all(g == pp.tolist() for g in gathered)
        if case == "powerlaw_int":
            x = hecgen.vector(A.n_cols, "int", seed=11)
        else:
            x = hecgen.vector(A.n_cols, "uniform", seed=11)
        a = plan.export(rank)
        x_loc = x[a.r0:a.r1].copy()
        halo = exchange_halo_host(plan, rank, x_loc)
        assert halo.tobytes() == x[a.recv_cols].tobytes()          # exact copy of the needed entries
        x_ext = np.concatenate([x_loc, halo])
        y_loc = np.empty(a.r1 - a.r0)
        for which, rows in ((hec.SUB_INTERIOR, a.interior), (hec.SUB_BOUNDARY, a.boundary)):
            M = plan.part_hec(A, rank, which, device=-1)
            e = M.export()
            R = H.HecRef(M.n_rows, M.n_cols, e.width, e.stride, e.ell_col, e.ell_val, e.tail_rows,
                         e.tail_ptr, e.tail_col, e.tail_val)
            y_loc[rows] = H.spmv(R, x_ext)
        y_ref = oracle.csr_spmv(A, x, a.r0, a.r1)
        tol = oracle.tolerance(A, x, a.r0, a.r1)
        ok = bool(np.all(np.abs(y_loc - y_ref) <= tol))
        if case == "powerlaw_int":
            ok = ok and y_loc.tobytes() == y_ref.tobytes()
        out_q.put((rank, ok, len(halo)))
    except Exception as ex:  # surface the failure to the parent
        out_q.put((rank, False, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "poisson"), (2, "powerlaw_int"), (3, "spe10"), (3, "powerlaw_int")])
def test_gloo_halo_exchange_and_partitioned_spmv(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in sorted(results, key=lambda t: t[0]):
        assert ok, f"rank {rank}: {info}"
    assert any(isinstance(info, int) and info > 0 for _, _, info in results)
