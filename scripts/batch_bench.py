"""Throughput of many small solves on one B200 (batch.solve_many): C1-sized
random_qp instances (2000 x 1000, sparse Q), sequential vs concurrent streams."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2602_23967_b200 as aq
from paper_2602_23967_b200 import batch

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
probs = [aq.random_qp(2000, 1000, "sparse", density=0.01, seed=s) for s in range(N)]
prm = aq.SolverParams(eps_tol=1e-8)
batch.solve_many(probs[:2], prm, streams=2)  # warm-up (module load, allocator)
out = {"instances": N, "workload": "random_qp(2000,1000,'sparse',0.01,seed) to 1e-8 (config 1 family)"}
for streams in (1, 4, 8, 16):
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = batch.solve_many(probs, prm, streams=streams)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    out[f"streams{streams}"] = {"seconds": round(dt, 3), "solves_per_s": round(N / dt, 2),
                                "solved": sum(r.status.value == "optimal" for r in res),
                                "outer_total": sum(r.outer_iterations for r in res)}
    print(json.dumps({streams: out[f"streams{streams}"]}), flush=True)
print(json.dumps(out))
