"""Executed warp instructions and stall samples of one kernel per CUDA source line / region.

    python tools/ncu_lines_by_region.py <report.ncu-rep> <object.o> <mangled kernel name> [top]

Reads the ncu source page (per SASS instruction) and maps every SASS address to its source line
(inlined-at line in fast.cuh when inlined) with nvdisasm -g of the object's cubin."""

import collections
import os
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def main():
    rep, obj, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    hdr = rows[1]
    ie, sp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[0], 16), int(r[ie] or 0), int(r[sp] or 0)) for r in rows[2:] if len(r) >= len(hdr)]
    base = data[0][0]
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=d, capture_output=True)
        cub = next(Path(d).glob("*.cubin"))
        dis = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout.splitlines()
    start = next(i for i, l in enumerate(dis) if l.startswith("//---") and fn in l)
    amap, cur = {}, None
    for l in dis[start + 1:]:
        if l.startswith("//---"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
        if m:
            inl = re.search(r'inlined at "([^"]+)", line (\d+)', m.group(3))
            if inl and not os.environ.get("INNER"):
                cur = (Path(inl.group(1)).name, int(inl.group(2)))
            else:
                cur = (Path(m.group(1)).name, int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            amap[int(m.group(1), 16)] = cur
    inst, samp = collections.Counter(), collections.Counter()
    for a, n, s in data:
        k = amap.get(a - base, ("?", 0))
        inst[k] += n
        samp[k] += s
    ti, ts = sum(inst.values()), max(sum(samp.values()), 1)
    print(f"total warp instructions {ti}, stall samples {ts}")
    import os
    order = samp if os.environ.get("SORT") == "samples" else inst
    for k, _ in order.most_common(top):
        v = inst[k]
        print(f"{k[0]}:{k[1]:5d}  inst {100 * v / ti:5.1f}%  samples {100 * samp[k] / ts:5.1f}%")


if __name__ == "__main__":
    main()
