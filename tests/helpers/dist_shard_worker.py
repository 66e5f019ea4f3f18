"""Worker of tests/test_gpu_dist.py (launched by torch.distributed.run): a
row-sharded solve through shard.DistGroup -- one process per rank, the
peers' solver workspaces mapped with CUDA IPC, exactly the multi-GPU path.
On a one-GPU box every rank shares cuda:0 (gloo for the host plumbing); the
contexts time-slice, so exchanges are slow, but every byte moves through the
real IPC mappings.  Rank 0 prints one JSON line per instance."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import instances  # noqa: E402  (instance specs only: the generators are the package's)
import paper_2602_23967_b200 as aq  # noqa: E402
from paper_2602_23967_b200.shard import DistGroup  # noqa: E402

ngpu = torch.cuda.device_count()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = rank % ngpu
torch.cuda.set_device(dev)
dist.init_process_group("nccl" if ngpu >= world else "gloo")
for spec, iters in (("c5:4e3:100:0", 192), ("rqp:300:150:low_rank:0.05:3", 128)):
    p = instances.build(spec)
    prm = aq.SolverParams(eps_tol=1e-8, iter_limit=iters)
    g = DistGroup()
    r = aq.solve(p, prm, device=dev, group=g)
    g.close()
    xs = [None] * world
    dist.all_gather_object(xs, (r.x.tobytes(), r.outer_iterations, r.inner_iterations))
    if rank == 0:
        one = aq.solve(p, prm, device=dev)
        same = all(x == xs[0] for x in xs)
        print(json.dumps({"spec": spec, "status": r.status.value, "outer": r.outer_iterations,
                          "inner": r.inner_iterations, "single_outer": one.outer_iterations,
                          "single_inner": one.inner_iterations, "ranks_identical": same,
                          "max_dx": float(np.abs(r.x - one.x).max()), "max_dy": float(np.abs(r.y - one.y).max()),
                          "scale": float(max(1.0, np.abs(one.x).max()))}), flush=True)
dist.destroy_process_group()
