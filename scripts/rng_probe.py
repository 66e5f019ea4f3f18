import os, sys, time, threading
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from paper_2602_23967_b200 import generators
from paper_2602_23967_b200.device import DeviceContext, DeviceProblem
print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for _ in range(2):
    t = time.perf_counter(); np.random.default_rng(0).standard_normal(50_000_000); print("rng alone", time.perf_counter() - t)
p = generators.banded_qp(50_000_000, 50_000_000, half_width=5000, seed=0)
ctx = DeviceContext.get(0)
d = DeviceProblem(p, ctx); del d; torch.cuda.synchronize()
for _ in range(2):
    res = {}
    def rng():
        t = time.perf_counter(); np.random.default_rng(0).standard_normal(50_000_000); res["rng"] = time.perf_counter() - t
    th = threading.Thread(target=rng); t0 = time.perf_counter(); th.start()
    d = DeviceProblem(p, ctx); torch.cuda.synchronize(); tu = time.perf_counter() - t0
    th.join(); print("concurrent: rng", res["rng"], "problem", tu); del d; torch.cuda.synchronize()
