"""Per-source-line warp-stall samples of one kernel from an ncu --set full capture (--import-source on), mapped
through nvdisasm line info of the object the kernel was built from (this container; the capture comes back from the
GPU box):   python tools/ncu_lines.py REPORT.ncu-rep OBJECT.o SOURCE.cu [N] [MANGLED_SUBSTRING]
(the substring picks the kernel's section when the object holds several kernels, e.g. k_assembleILi0ELb0E)"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def main():
    rep, obj, src = sys.argv[1:4]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    fn = sys.argv[5] if len(sys.argv) > 5 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    data = rows[2:]
    iS = h.index("Warp Stall Sampling (All Samples)")
    iE = h.index("Instructions Executed")
    base = int(data[0][0], 16)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, stdout=subprocess.DEVNULL,
                       stderr=subprocess.DEVNULL)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], stdout=subprocess.PIPE,
                              stderr=subprocess.DEVNULL, text=True).stdout
    line, off2line, inside = None, {}, not fn
    for l in sass.splitlines():
        if l.startswith(".text."):
            inside = not fn or fn in l
        if not inside:
            continue
        m = re.search(r"line (\d+)", l)
        if m:
            line = int(m.group(1))
        m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m2:
            off2line[int(m2.group(1), 16)] = line
    agg = defaultdict(lambda: [0, 0])
    tot_s = tot_e = 0
    for r in data:
        if not r[iS].isdigit():
            continue
        s, e = int(r[iS]), int(r[iE]) if r[iE].isdigit() else 0
        tot_s += s
        tot_e += e
        ln = off2line.get(int(r[0], 16) - base)
        agg[ln][0] += s
        agg[ln][1] += e
    text = open(src).read().split("\n")
    print(f"samples {tot_s}  warp instructions {tot_e}")
    for ln, (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
        t = text[ln - 1].strip()[:90] if ln else "?"
        print(f"{s:7d} {100 * s / tot_s:5.1f}% {e:10d} {ln} {t}")


if __name__ == "__main__":
    main()
