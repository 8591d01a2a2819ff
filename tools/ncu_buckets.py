"""Stall samples / executed instructions of one kernel per 8 KB SASS address bucket, with the
source lines (file:line, innermost) most frequent in each bucket.

    python tools/ncu_buckets.py <report.ncu-rep> <object.o> <mangled kernel name>"""

import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path


def main():
    rep, obj, fn = sys.argv[1:4]
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    base = int(data[0][0], 16)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=d, capture_output=True)
        cub = next(Path(d).glob("*.cubin"))
        dis = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout.splitlines()
    start = next(i for i, l in enumerate(dis) if l.startswith("//---") and fn in l)
    cur, amap = None, {}
    for l in dis[start + 1:]:
        if l.startswith("//---"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = Path(m.group(1)).name + ":" + m.group(2)
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            amap[int(m.group(1), 16)] = cur
    b, bi = collections.Counter(), collections.Counter()
    lines = collections.defaultdict(collections.Counter)
    tot = max(sum(int(r[si] or 0) for r in data), 1)
    toti = max(sum(int(r[ie] or 0) for r in data), 1)
    for r in data:
        a = int(r[0], 16) - base
        k = a // 0x2000
        b[k] += int(r[si] or 0)
        bi[k] += int(r[ie] or 0)
        c = amap.get(a)
        if c and not c.startswith("sm_") and not c.startswith("device_"):
            lines[k][c] += int(r[si] or 0) + 1
    for k in sorted(b):
        if b[k] / tot > 0.01 or bi[k] / toti > 0.01:
            print(f"{k * 0x2000:#07x} samples {100 * b[k] / tot:5.1f}% inst {100 * bi[k] / toti:5.1f}%  "
                  + " ".join(x for x, _ in lines[k].most_common(5)))


if __name__ == "__main__":
    main()
