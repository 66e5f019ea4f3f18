"""Round-2 profiling digests into profiles/ (committed evidence):

* ``launch_share_r02.txt``: the ncu launch list of the bench command itself
  (eager mode, gpu__time_duration per launch): per-kernel count, time, share;
* ``ncu_summary_r02.json``: per-kernel digest of the stand-alone --set full
  captures of scripts/profile_r02.sh (C5 and C2 hot kernels): duration, DRAM
  bytes per launch against the algorithmic bytes, throughputs, occupancy,
  top stall reasons.

    python scripts/summarize_r02.py
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"  # r02: tile kernels; r02e: banded ring path
sys.argv = [sys.argv[0], TAG, os.path.join(ROOT, "profiles")]
import summarize_profiles as sp  # noqa: E402  (reuses digest / short)

OUT = os.path.join(ROOT, "profiles")
# kernel name -> role (the stand-alone launches of scripts/prof_kernel.py <cfg> 0,1,2,3,4,5)
ROLES = [("spmv_op<OpGrad<0>", "bb_gradient"), ("spmv_ring_op<OpGrad<0>", "bb_gradient"),
         ("spmv_ring_op<OpP2", "p2_A_xbar"), ("k_step2", "bb_step"), ("OpP1Bb", "p1_At_y"),
         ("spmv_op<OpP2", "p2_A_xbar"), ("elem_op<OpXPost", "x_post"), ("fin_ctrl_cl<OpGrad", "bb_fold"),
         ("fin_ctrl_cl<OpP2", "p2_fold"), ("fin_ctrl_cl<OpXPost", "x_fold")]
# algorithmic bytes (SURVEY.md §8(d) pass model; bench.kernel_table)
ALG = {
    "c5": {"bb_gradient": 6399975980, "bb_step": 2000000000, "p1_At_y": 8597110104, "p2_A_xbar": 8997110104,
           "x_post": 2400000000},
    "c2": {"bb_gradient": 128000000 - 4 + 4, "bb_step": 40000000, "p1_At_y": 96000004, "p2_A_xbar": 82000004,
           "x_post": 48000000},
}


def launch_share():
    path = os.path.join(ROOT, "gpurun_out", f"launches_{TAG}.csv")
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    agg = collections.defaultdict(lambda: {"n": 0, "ns": 0.0})
    for r in csv.DictReader(lines[start:]):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = sp.short(r["Kernel Name"])
        agg[k]["n"] += 1
        agg[k]["ns"] += float(r["Metric Value"].replace(",", "")) * (1e3 if r["Metric Unit"] == "usecond" else
                                                                      (1e6 if r["Metric Unit"] == "msecond" else 1))
    tot = sum(a["ns"] for a in agg.values())
    with open(os.path.join(OUT, f"launch_share_{TAG}.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 3000, of\n")
        f.write("#   AQP_EAGER=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline (C5 headline command;\n")
        f.write("#   eager mode: ncu cannot profile kernel nodes of graphs with conditional nodes)\n")
        f.write("# every launch of the process (setup, power iteration, 5 outer iterations, checks, kernel table);\n")
        f.write("# cold-cache serialised launches: compare SHARES, not absolute times\n")
        f.write(f"{'kernel':48s} {'launches':>8s} {'total_ms':>10s} {'share':>6s} {'avg_us':>9s}\n")
        for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
            f.write(f"{k:48s} {a['n']:8d} {a['ns'] / 1e6:10.2f} {100 * a['ns'] / tot:5.1f}% {a['ns'] / a['n'] / 1e3:9.1f}\n")
    print(open(os.path.join(OUT, f"launch_share_{TAG}.txt")).read())


def main():
    launch_share()
    summary = {"tag": TAG, "note": "ncu --set full --clock-control none --import-source on; stand-alone launches "
               "(scripts/prof_kernel.py <cfg> 0,1,2,3,4,5, each after an L2 flush); alg_bytes: SURVEY.md §8(d)",
               "kernels": {}}
    for cfg in ("c5", "c2"):
        rep = os.path.join(ROOT, "gpurun_out", "ncu", f"{cfg}_{TAG}.ncu-rep")
        for dg in sp.digest(rep):
            name = next((r for pat, r in ROLES if pat in dg["kernel"]), None)
            if name is None or f"{cfg}_{name}" in summary["kernels"]:
                continue
            alg = ALG[cfg].get(name)
            if alg:
                dg["alg_bytes"] = alg
                dg["dram_over_alg"] = round(dg["dram_bytes_per_launch"] / alg, 3)
            summary["kernels"][f"{cfg}_{name}"] = dg
    with open(os.path.join(OUT, f"ncu_summary_{TAG}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    for k, v in summary["kernels"].items():
        print(k, v["kernel"], v["details"].get("Duration"), v["details"].get("DRAM Throughput"), v.get("dram_over_alg"))


if __name__ == "__main__":
    main()
