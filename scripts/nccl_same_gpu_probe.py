"""Probe: can two NCCL ranks share ONE GPU (two processes, both on cuda:0)?
If NCCL accepts it, the NCCL send/recv halo branch of hec_spmv_dist can be
exercised with a real peer on a one-GPU box.  Prints one line per rank."""
import os, sys, socket, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "RANK" not in os.environ:
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    procs = [subprocess.Popen([sys.executable, __file__], env=dict(os.environ, RANK=str(r), WORLD_SIZE="2",
             MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_DEBUG="WARN")) for r in range(2)]
    sys.exit(max(p.wait() for p in procs))
sys.path.insert(0, ROOT)
import numpy as np, torch, torch.distributed as dist
import hecgen, oracle
import paper_1606_00545_b200 as hec
rank = int(os.environ["RANK"])
dist.init_process_group("gloo", rank=rank, world_size=2)
torch.cuda.set_device(0)
A = hecgen.poisson3d(48, 40, 32)
plan = hec.partition(A, 2, hec.PART_GRID, (48, 40, 32))
obj = [hec.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
try:
    D = hec.Dist(A, plan, rank, obj[0], 0)
except Exception as e:
    print(f"rank {rank}: NCCL communicator on a shared GPU refused: {e}", flush=True)
    sys.exit(0)
pp = plan.part_ptr(); r0, r1 = int(pp[rank]), int(pp[rank + 1])
bad = 0
for it in range(4):
    x = hecgen.vector(A.n_cols, "uniform", seed=50 + it)
    xl = torch.from_numpy(np.ascontiguousarray(x[r0:r1])).cuda()
    yl = torch.full((r1 - r0,), float("nan"), dtype=torch.float64, device="cuda")
    D.spmv(xl, yl)
    torch.cuda.synchronize()
    ok = np.abs(yl.cpu().numpy() - oracle.csr_spmv(A, x, r0, r1)) <= oracle.tolerance(A, x, r0, r1)
    bad += int((~ok).sum())
print(f"rank {rank}: NCCL send/recv halo with a real peer on a shared GPU: bad rows {bad}", flush=True)
dist.barrier()
D.free()
sys.exit(1 if bad else 0)
