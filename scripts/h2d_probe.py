"""H2D upload strategies for multi-GB numpy arrays (design probe for the e2e path).

    python scripts/h2d_probe.py [GB]
"""

from __future__ import annotations

import concurrent.futures as cf
import json
import os
import sys
import time

import numpy as np
import torch


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t


def main():
    gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    n = int(gb * 2**30 / 8)
    a = np.random.default_rng(0).random(n)
    dst = torch.empty(n, dtype=torch.float64, device="cuda")
    out = {"gb": gb, "nproc": os.cpu_count()}
    out["pageable_to"] = gb / timed(lambda: dst.copy_(torch.from_numpy(a)))
    rt = torch.cuda.cudart()

    def reg():
        rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        dst.copy_(torch.from_numpy(a), non_blocking=True)
        torch.cuda.synchronize()
        rt.cudaHostUnregister(a.ctypes.data)

    t_reg = timed(lambda: rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0))
    t_cp = timed(lambda: dst.copy_(torch.from_numpy(a), non_blocking=True))
    t_unreg = timed(lambda: rt.cudaHostUnregister(a.ctypes.data))
    out["register_s"], out["registered_copy_gbs"], out["unregister_s"] = t_reg, gb / t_cp, t_unreg
    out["register_total_gbs"] = gb / (t_reg + t_cp + t_unreg)
    for threads, chunk_mb in ((4, 32), (8, 32), (8, 64), (16, 16), (16, 32)):
        chunk = chunk_mb * 2**20 // 8
        bufs = [[torch.empty(chunk, dtype=torch.float64).pin_memory() for _ in range(2)] for _ in range(threads)]
        streams = [torch.cuda.Stream() for _ in range(threads)]
        evs = [[None, None] for _ in range(threads)]
        nch = (n + chunk - 1) // chunk

        def worker(t):
            s = streams[t]
            j = 0
            for c in range(t, nch, threads):
                b = bufs[t][j & 1]
                if evs[t][j & 1] is not None:
                    evs[t][j & 1].synchronize()
                lo, hi = c * chunk, min(n, (c + 1) * chunk)
                np.copyto(b.numpy()[: hi - lo], a[lo:hi])
                with torch.cuda.stream(s):
                    dst[lo:hi].copy_(b[: hi - lo], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(s)
                evs[t][j & 1] = e
                j += 1
            s.synchronize()

        def run():
            with cf.ThreadPoolExecutor(threads) as ex:
                list(ex.map(worker, range(threads)))

        run()
        out[f"staged_t{threads}_c{chunk_mb}"] = gb / timed(run)
        del bufs
    ok = torch.equal(dst.cpu(), torch.from_numpy(a))
    out["ok"] = bool(ok)
    # D2H for comparison
    h = np.empty(n)
    out["d2h_pageable"] = gb / timed(lambda: torch.from_numpy(h).copy_(dst))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
