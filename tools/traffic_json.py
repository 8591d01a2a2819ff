"""profiles/fast_kernel_traffic.json from an ncu launch list with dram__bytes_read/write.sum
(tools/gpu_final.sh: the bench step, C2 x1.0): DRAM bytes of the single pass per launch (the last
fast_scan_kernel + fast_kernel launch pair), against the trace's algorithmic bytes.

    python tools/traffic_json.py <launches.csv> <source label>"""

import csv
import json
import sys
from pathlib import Path

ALGO = 3210383245  # C2 x1.0 trace bytes (bench.py workload_detail.bytes_per_gpu_rank0)


def main():
    path, label = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        name = r[ki]
        if "fast_kernel<" in name or "fast_scan_kernel" in name:
            per.setdefault((int(r[ii]), "scan" if "fast_scan" in name else "main"), {})[r[mi]] = float(r[vi].replace(",", ""))
    last_main = max(i for i, k in per if k == "main")
    scan = [i for i, k in per if k == "scan" and i < last_main]
    m = per[(last_main, "main")]
    s = per[(max(scan), "scan")] if scan else {}
    rd = m["dram__bytes_read.sum"] + s.get("dram__bytes_read.sum", 0)
    wr = m["dram__bytes_write.sum"] + s.get("dram__bytes_write.sum", 0)
    out = {"kernel": "fast_scan_kernel + fast_kernel" if scan else "fast_kernel", "dram_read": int(rd),
           "dram_write": int(wr), "dram_bytes_per_launch": int(rd + wr), "algorithmic_bytes": ALGO,
           "ratio": (rd + wr) / ALGO, "source": label}
    Path("profiles/fast_kernel_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
