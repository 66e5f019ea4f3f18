"""torchrun --nproc-per-node 2: DistGroup (CUDA IPC) row-sharded solve.  On a
1-GPU box both ranks share cuda:0 (gloo for the plumbing; the contexts
time-slice, so exchanges are slow but the IPC path is exercised)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import torch.distributed as dist
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200.shard import DistGroup

ngpu = torch.cuda.device_count()
rank = int(os.environ["RANK"])
dev = rank % ngpu
torch.cuda.set_device(dev)
dist.init_process_group("nccl" if ngpu >= int(os.environ["WORLD_SIZE"]) else "gloo")
p = aq.random_qp(300, 150, "sparse", density=0.05, seed=7)
prm = aq.SolverParams(eps_tol=1e-8, iter_limit=int(os.environ.get("ITERS", "128")))
t = time.time()
g = DistGroup()
r = aq.solve(p, prm, device=dev, group=g)
one = aq.solve(p, prm, device=dev) if rank == 0 else None
if rank == 0:
    print(f"dist P={g.nranks}: {r.status.value} outer={r.outer_iterations} inner={r.inner_iterations} "
          f"({time.time()-t:.1f}s) max|x-x1|={np.abs(r.x-one.x).max():.3e} single={one.status.value} "
          f"outer={one.outer_iterations} inner={one.inner_iterations}", flush=True)
g.close()
dist.destroy_process_group()
