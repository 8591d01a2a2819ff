"""Instruction share per source function of one kernel in an ncu report.

    python tools/ncu_funcs.py <report.ncu-rep> <kernel-regex>"""

import collections
import csv
import re
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          "regex:" + kern], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, cur_line = "?", 0
    inst = collections.Counter()
    tot = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No", "Kernel Name"):
            continue
        if r[0] != "":
            cur_line = int(r[0]) if r[0].isdigit() else 0
            continue
        if len(r) > 7 and r[2].startswith("0x"):
            try:
                n = int(r[7])
            except ValueError:
                continue
            inst[(cur_file, cur_line)] += n
            tot += n
    starts = {}
    for f in {f for f, _ in inst}:
        try:
            src = open(f"paper_2504_03683_b200/csrc/{f}").read().splitlines()
        except OSError:
            continue
        st = []
        for i, line in enumerate(src, 1):
            m = re.match(r"^(?:__device__|__global__|template|static|__host__|struct)[^(]*?(\w+)\s*[({]", line)
            if m:
                st.append((i, m.group(1)))
        starts[f] = st
    res = collections.Counter()
    for (f, ln), n in inst.items():
        name = "?"
        for a, nm in starts.get(f, []):
            if a <= ln:
                name = nm
        res[f"{f}:{name}"] += n
    print(f"total instructions {tot}")
    for k, n in res.most_common(30):
        print(f"{k:45s} {100 * n / tot:6.2f}")


if __name__ == "__main__":
    main()
