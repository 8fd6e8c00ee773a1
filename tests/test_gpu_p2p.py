"""GPU parity of the peer-memory halo transport: the fused push
kernel (pack + stores into the destination rank's window + epoch release),
the flag wait and the boundary rows as its programmatic dependent.

- One process, all ranks on one device (hec_dist_p2p_connect_local): many
  consecutive calls with fresh x (the windows alternate by call parity),
  compared with the copy-based emulation (bitwise: same kernels, same data)
  and with the oracle (tolerance; bitwise on integer data).
- Two processes sharing the one GPU through CUDA IPC (hec_dist_create_p2p +
  handles all-gathered over a gloo group + hec_dist_p2p_connect): the real
  multi-process path, with the two ranks' kernels time-sliced on one device."""
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import hecgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1606_00545_b200 as hec  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def local_calls(A, xs_full, P, kind, grid=None, p2p=True):
    plan = hec.partition(A, P, kind, grid)
    grp = hec.LocalDistGroup(A, plan, 0, None, p2p=p2p)
    pp = plan.part_ptr()
    outs = []
    for x in xs_full:  # consecutive calls: epochs 1, 2, 3, ... (both buffer parities)
        xs = [torch.from_numpy(np.ascontiguousarray(x[pp[p]:pp[p + 1]])).cuda() for p in range(P)]
        ys = [torch.full((int(pp[p + 1] - pp[p]),), float("nan"), dtype=torch.float64, device="cuda")
              for p in range(P)]
        grp.spmv(xs, ys)
        torch.cuda.synchronize()
        outs.append(np.concatenate([t.cpu().numpy() for t in ys]))
    for r in grp.ranks:
        r.check()
    launches = [r.info.launches for r in grp.ranks]
    grp.free()
    return outs, launches


CASES = [
    ("poisson_slabs", lambda: hecgen.poisson3d(32, 24, 16), hec.PART_GRID, (32, 24, 16), [2, 3, 4, 8]),
    ("powerlaw_nnz", lambda: hecgen.powerlaw(1 << 15, seed=5), hec.PART_CONTIG_NNZ, None, [2, 4, 8]),
    ("spe10_nnz", lambda: hecgen.spe10(20, 30, 10, seed=3), hec.PART_CONTIG_NNZ, None, [3, 5]),
    # nonsymmetric pattern: some ranks send to a neighbour they receive nothing from
    ("random_nonsym", lambda: hecgen.random_csr(300, 300, 0.01, seed=7), hec.PART_CONTIG_ROWS, None, [4, 7]),
]


@pytest.mark.parametrize("name,maker,kind,grid,Ps", CASES)
def test_local_p2p_matches_copy_emulation_and_oracle(name, maker, kind, grid, Ps):
    A = maker()
    xs = [hecgen.vector(A.n_cols, "uniform", seed=s) for s in (1, 2, 3, 4, 5)]
    for P in Ps:
        got, launches = local_calls(A, xs, P, kind, grid, p2p=True)
        ref_copy, _ = local_calls(A, xs, P, kind, grid, p2p=False)
        for x, y, yc in zip(xs, got, ref_copy):
            assert y.tobytes() == yc.tobytes()
            assert np.all(np.abs(y - oracle.csr_spmv(A, x)) <= oracle.tolerance(A, x))
        assert max(launches) >= 3  # push + wait + at least one product kernel on some rank


def test_local_p2p_integer_bitwise_many_calls():
    A = hecgen.powerlaw(1 << 14, integer_values=True, seed=9)
    xs = [hecgen.vector(A.n_cols, "int", seed=s) for s in range(7)]
    got, _ = local_calls(A, xs, 6, hec.PART_CONTIG_NNZ)
    for x, y in zip(xs, got):
        assert y.tobytes() == oracle.csr_spmv(A, x).tobytes()


def test_local_p2p_every_row_its_own_part():
    B = hecgen.random_csr(24, 24, 0.2, seed=1)
    xs = [hecgen.vector(24, "uniform", seed=s) for s in (1, 2, 3)]
    got, _ = local_calls(B, xs, 24, hec.PART_CONTIG_ROWS)
    for x, y in zip(xs, got):
        assert np.all(np.abs(y - oracle.csr_spmv(B, x)) <= oracle.tolerance(B, x))


def test_p2p_handle_without_transport_is_refused():
    A = hecgen.poisson2d(16, 16)
    plan = hec.partition(A, 2, hec.PART_CONTIG_ROWS)
    D, h = hec.Dist.create_p2p(A, plan, 0, 0)
    assert len(h) == hec.IPC_BYTES
    x = torch.zeros(D.n_loc, dtype=torch.float64, device="cuda")
    y = torch.zeros(D.n_loc, dtype=torch.float64, device="cuda")
    with pytest.raises(hec.HecError) as e:
        D.spmv(x, y)        # not connected: no halo transport
    assert e.value.status == 8
    with pytest.raises(hec.HecError) as e:
        D.cg(x, y, 1e-8, 5)  # no NCCL communicator for the dot products
    assert e.value.status == 8
    D.free()


WORKER = textwrap.dedent(r"""
    import os, sys, numpy as np, torch, torch.distributed as dist
    sys.path.insert(0, os.environ["HEC_ROOT"])
    import hecgen, oracle
    import paper_1606_00545_b200 as hec
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = os.environ["HEC_CASE"]
    if cfg == "slabs":
        A = hecgen.poisson3d(48, 40, 32); plan = hec.partition(A, world, hec.PART_GRID, (48, 40, 32))
    elif cfg == "slabs256":   # BASELINE configs[2] at full size, every row of each rank
        A = hecgen.poisson3d(256, 256, 256); plan = hec.partition(A, world, hec.PART_GRID, (256, 256, 256))
    else:
        A = hecgen.powerlaw(1 << 15, seed=3); plan = hec.partition(A, world, hec.PART_CONTIG_NNZ)
    D, h = hec.Dist.create_p2p(A, plan, rank, 0)
    hs = [None] * world
    dist.all_gather_object(hs, h)
    D.p2p_connect(hs)
    pp = plan.part_ptr(); r0, r1 = int(pp[rank]), int(pp[rank + 1])
    bad = 0
    for it in range(6 if cfg != "slabs256" else 2):
        x = hecgen.vector(A.n_cols, "uniform", seed=100 + it)
        xl = torch.from_numpy(np.ascontiguousarray(x[r0:r1])).cuda()
        yl = torch.full((r1 - r0,), float("nan"), dtype=torch.float64, device="cuda")
        D.spmv(xl, yl)
        torch.cuda.synchronize()
        y = yl.cpu().numpy()
        ok = np.abs(y - oracle.csr_spmv(A, x, r0, r1)) <= oracle.tolerance(A, x, r0, r1)
        bad += int((~ok).sum())
    D.check()
    # phase timing (the overlap evidence): both ends of the last call
    D.set_timing(True)
    xl = torch.from_numpy(np.ascontiguousarray(hecgen.vector(A.n_cols, "uniform", seed=99)[r0:r1])).cuda()
    D.spmv(xl, yl)
    t_int, t_comm = D.phase_times()
    D.set_timing(False)
    if not (t_int > 0 and t_comm > 0):
        bad += 1
    print(f"rank {rank} launches {D.info.launches} bad {bad} interior {t_int:.4f} ms comm {t_comm:.4f} ms", flush=True)
    dist.barrier()
    D.free()
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)
""")


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("case,world", [("slabs", 2), ("powerlaw", 2), ("slabs", 3), ("slabs256", 2)])
def test_two_processes_one_gpu_ipc(tmp_path, case, world):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), HEC_ROOT=ROOT, HEC_CASE=case)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=500)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for p, out in zip(procs, outs):
        assert p.returncode == 0, out[-3000:]
        assert "bad 0" in out
