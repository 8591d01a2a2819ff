"""Summarise ncu captures into the text files committed under profiles/.

    python tools/ncu_summary.py full  <report.ncu-rep>   # --set full capture of one tile_kernel launch
    python tools/ncu_summary.py launches <launches.csv>  # --metrics gpu__time_duration.sum launch list
"""

import collections
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Achieved Active Warps Per SM",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
        "No Eligible", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum"]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    print(f"# ncu --set full: {rep}")
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEYS:
            print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, u, v = rr[0], rr[1], rr[2]
    for i, n in enumerate(h):
        if n in RAW:
            print(f"{n:40s} {v[i]} {u[i]}")
    print("# warp stall samples (all)")
    stalls = []
    for i, n in enumerate(h):
        if "smsp__pcsamp_warps_issue_stalled" in n and "not_issued" not in n:
            try:
                stalls.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    for s, n in sorted(stalls, reverse=True)[:10]:
        print(f"  {n:28s} {s / tot * 100:5.1f}%")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    tot, n = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0]
            tot[k] += float(d["Metric Value"])
            n[k] += 1
    t = sum(tot.values())
    print(f"# launch list {path} (ncu, cold cache, serialised: compare shares)")
    for k, v in tot.most_common():
        print(f"{k:40s} launches={n[k]:3d} avg={v / n[k] / 1e6:8.3f} ms share={v / t * 100:5.1f}%")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
