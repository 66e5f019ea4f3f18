"""Summarise gpurun_out/ ncu captures (scripts/profile_round.sh) into profiles/
(committed evidence): the launch-share table of one eager C2 window and a
per-kernel digest of every --set full report (duration, DRAM bytes per launch,
throughputs, occupancy, top stall reasons).

    python scripts/summarize_profiles.py r01
"""
import collections, csv, glob, json, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
OUT = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles")
os.makedirs(OUT, exist_ok=True)
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    m = re.search(r"aqp::(\w+)<aqp::(Op\w+(?:<\(bool\)\d>)?)(?:, \(bool\)(\d))?", name)
    if m:
        return f"{m.group(1)}<{m.group(2)}{',uniform' if m.group(3) == '1' else ''}>"
    m = re.search(r"aqp::(\w+)", name)
    return m.group(1) if m else name[:40]


def launch_share():
    path = os.path.join(ROOT, "gpurun_out", "launches.csv")
    if not os.path.exists(path):
        return
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    agg = collections.defaultdict(lambda: {"n": 0, "ns": 0.0, "dram": 0.0})
    for r in csv.DictReader(lines[start:]):
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            agg[k]["n"] += 1
            agg[k]["ns"] += v
        else:
            agg[k]["dram"] += v * SCALE.get(r["Metric Unit"], 1)
    tot = sum(a["ns"] for a in agg.values())
    rows = sorted(agg.items(), key=lambda kv: -kv[1]["ns"])
    with open(os.path.join(OUT, f"{tag}_launch_share.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_{read,write}.sum --clock-control none\n")
        f.write("# one C2 certification window (64 outer iterations) in eager mode (AQP_EAGER=1),\n")
        f.write("# cold-cache serialised launches: compare SHARES, not absolute times\n")
        f.write(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s} {'dram_MB/launch':>14s}\n")
        for k, a in rows:
            f.write(f"{k:44s} {a['n']:8d} {a['ns']/1e3:10.1f} {100*a['ns']/tot:5.1f}% "
                    f"{a['ns']/a['n']/1e3:8.2f} {a['dram']/a['n']/1e6:14.2f}\n")
    print(open(os.path.join(OUT, f"{tag}_launch_share.txt")).read())


KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "Issue Slots Busy", "Eligible Warps Per Scheduler", "Grid Size",
        "Block Size", "Waves Per SM"]


def digest(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hdr, units = rr[0], rr[1]
    out = []
    dets = collections.defaultdict(dict)
    rws = list(csv.reader(det.splitlines()))
    ix = {h: i for i, h in enumerate(rws[0])}
    for r in rws[1:]:
        dets[r[ix["ID"]]][r[ix["Metric Name"]]] = f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]}".strip()
    for row in rr[2:]:
        vals = dict(zip(hdr, row))
        u = dict(zip(hdr, units))

        def num(k):
            try:
                return float(vals[k].replace(",", "")) * SCALE.get(u.get(k, "byte"), 1)
            except Exception:
                return None

        stalls = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), num(k) or 0) for k in vals
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")),
                        key=lambda kv: -kv[1])[:8]
        rd, wr = num("dram__bytes_read.sum") or 0.0, num("dram__bytes_write.sum") or 0.0
        d = dets.get(vals.get("ID"), {})
        out.append({"kernel": short(vals.get("Kernel Name", "")), "dram_bytes_per_launch": rd + wr,
                    "dram_read": rd, "dram_write": wr, "details": {k: d[k] for k in KEEP if k in d},
                    "top_stalls": dict(stalls)})
    return out


if __name__ == "__main__":
    launch_share()
    names = {"c2_bb_gradient": ["bb_gradient"], "c2_bb_step": ["bb_step"], "c2_bb_fold": ["bb_fold"],
             "c2_p1": ["c2_p1_At_y"], "c2_p2": ["c2_p2_A_xbar"],
             "c5_passes": ["c5_bb_gradient", "c5_p1_At_y", "c5_p2_A_xbar"], "c3_dense": ["c3_dense_Rx", "c3_dense_Rtv"]}
    summary = {"tag": tag, "note": "ncu --set full --clock-control none; one launch per kernel; C2 from an eager "
               "window (scripts/prof_c2.py), C5/C3 stand-alone launches (scripts/prof_kernel.py)", "kernels": {}}
    for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "ncu", "*.ncu-rep"))):
        base = os.path.basename(rep)[:-8]
        if base not in names:
            continue
        for key, dg in zip(names[base], digest(rep)):
            summary["kernels"][key] = dg
    with open(os.path.join(OUT, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: (v["kernel"], v["details"].get("Duration"), v["details"].get("DRAM Throughput"))
                      for k, v in summary["kernels"].items()}, indent=1))
