"""Summarise gpurun_out/ ncu captures into profiles/ (committed evidence)."""
import collections, csv, json, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

def short(name):
    m = re.search(r"aqp::(\w+)<aqp::(Op\w+(?:<\(bool\)\d>)?)(?:, \(bool\)(\d))?", name)
    if m:
        return f"{m.group(1)}<{m.group(2)}{',uniform' if m.group(3) == '1' else ''}>"
    m = re.search(r"aqp::(\w+)", name)
    return m.group(1) if m else name[:40]

lines = open(os.path.join(ROOT, "gpurun_out", "launches.csv")).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
agg = collections.defaultdict(lambda: {"n": 0, "ns": 0.0, "dram": 0.0})
for r in csv.DictReader(lines[start:]):
    k = short(r["Kernel Name"])
    v = float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        agg[k]["n"] += 1
        agg[k]["ns"] += v
    else:
        agg[k]["dram"] += v * (1e6 if r["Metric Unit"] == "Mbyte" else 1e9 if r["Metric Unit"] == "Gbyte" else 1e3 if r["Metric Unit"] == "Kbyte" else 1)
tot = sum(a["ns"] for a in agg.values())
rows = sorted(agg.items(), key=lambda kv: -kv[1]["ns"])
with open(os.path.join(OUT, f"{tag}_launch_share.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_{read,write}.sum --clock-control none\n")
    f.write("# one C2 certification window (64 outer iterations) in eager mode (AQP_EAGER=1),\n")
    f.write("# cold-cache serialised launches: compare SHARES, not absolute times\n")
    f.write(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s} {'dram_MB/launch':>14s}\n")
    for k, a in rows:
        f.write(f"{k:44s} {a['n']:8d} {a['ns']/1e3:10.1f} {100*a['ns']/tot:5.1f}% {a['ns']/a['n']/1e3:8.2f} {a['dram']/a['n']/1e6:14.2f}\n")
print(open(os.path.join(OUT, f"{tag}_launch_share.txt")).read())

def ncu_details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rws = list(csv.reader(out.splitlines()))
    hdr = rws[0]; ix = {h: i for i, h in enumerate(hdr)}
    d = {}
    for r in rws[1:]:
        if r[ix["ID"]] != "0":
            continue
        d[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    vals = dict(zip(rr[0], rr[2]))
    return d, vals

summary = {"tag": tag, "kernels": {}}
for name, rep in (("bb_gradient", "prof_grad"), ("bb_step", "prof_step")):
    path = os.path.join(ROOT, "gpurun_out", rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    d, vals = ncu_details(path)
    def num(k):
        try:
            return float(vals[k].replace(",", ""))
        except Exception:
            return None
    unit = (vals.get("dram__bytes_read.sum") or "")
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    units = dict(zip(*list(csv.reader(subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()))[:2]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rdb = rd * scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
    wrb = wr * scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
    stalls = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), num(k) or 0) for k in vals
                     if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")), key=lambda kv: -kv[1])[:8]
    keep = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
            "Issue Slots Busy", "Eligible Warps Per Scheduler", "Grid Size", "Waves Per SM"]
    summary["kernels"][name] = {
        "dram_bytes_per_launch": rdb + wrb, "dram_read": rdb, "dram_write": wrb,
        "details": {k: " ".join(d[k]) for k in keep if k in d},
        "top_stalls": dict(stalls),
    }
with open(os.path.join(OUT, "ncu_summary.json"), "w") as f:
    json.dump(summary, f, indent=1)
print(json.dumps(summary, indent=1))
