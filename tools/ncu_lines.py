"""Per-source-line instruction and stall-sample totals from an ncu report.

    python tools/ncu_lines.py <report.ncu-rep> [top] [kernel-regex]

Aggregates the SASS rows of `ncu --page source --print-source cuda,sass` under
the CUDA line they belong to (inlined code counts at its own file:line)."""

import collections
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if len(sys.argv) > 3:
        cmd += ["-k", "regex:" + sys.argv[3]]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, cur_line = "?", "?"
    inst = collections.Counter()
    samp = collections.Counter()
    total_i = total_s = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No", "Kernel Name"):
            continue
        if r[0] != "":
            cur_line = r[0]
            continue
        if len(r) > 7 and r[2].startswith("0x"):
            try:
                n = int(r[7])
                s = int(r[4])
            except ValueError:
                continue
            inst[(cur_file, cur_line)] += n
            samp[(cur_file, cur_line)] += s
            total_i += n
            total_s += s
    src = {}
    print(f"total instructions {total_i}, stall samples {total_s}")
    print(f"{'file:line':28s} {'inst%':>6s} {'samp%':>6s}  source")
    key = (lambda kv: samp[kv[0]]) if "--by-samples" in sys.argv else (lambda kv: kv[1])
    for (f, ln), n in sorted(inst.items(), key=key, reverse=True)[:top]:
        if f not in src:
            try:
                src[f] = open(f"paper_2504_03683_b200/csrc/{f}").read().splitlines()
            except OSError:
                src[f] = []
        text = src[f][int(ln) - 1].strip() if ln.isdigit() and int(ln) <= len(src[f]) else ""
        print(f"{f + ':' + ln:28s} {100 * n / total_i:6.2f} {100 * samp[(f, ln)] / max(total_s, 1):6.2f}  {text[:90]}")


if __name__ == "__main__":
    main()
