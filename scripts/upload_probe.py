"""aqp_h2d / aqp_d2h throughput on multi-GB arrays (design probe).

    python scripts/upload_probe.py [GB]
"""
import ctypes as C
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_23967_b200.device import DeviceContext  # noqa: E402

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
a = np.random.default_rng(0).random(int(gb * 2**30 / 8))
ctx = DeviceContext.get(0)
out = {}
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d = ctx.upload(a)
    torch.cuda.synchronize()
    out[f"h2d_{rep}"] = gb / (time.perf_counter() - t)
    del d
# with a concurrent host RNG draw (what solve() does during the upload)
th = threading.Thread(target=lambda: np.random.default_rng(0).standard_normal(50_000_000))
th.start()
t = time.perf_counter()
d = ctx.upload(a)
torch.cuda.synchronize()
out["h2d_with_rng"] = gb / (time.perf_counter() - t)
th.join()
back = np.empty_like(a)
for rep in range(2):
    t = time.perf_counter()
    ctx.lib.aqp_d2h(ctx.handle, C.c_void_p(back.ctypes.data), C.c_void_p(d.data_ptr()), a.nbytes)
    out[f"d2h_{rep}"] = gb / (time.perf_counter() - t)
out["ok"] = bool(np.array_equal(back, a))
print(json.dumps(out))
