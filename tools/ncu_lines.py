"""Per-source-line totals of an ncu --page source (SASS) export, joined with
the cubin's line table: L2 sectors, excessive sectors, stall samples.
usage: ncu_lines.py <rep> <cubin> <kernel-substring> [top]"""
import collections
import csv
import re
import subprocess
import sys

rep, cubin, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout.splitlines()
st = [i for i, l in enumerate(sass) if kname in l and l.strip().startswith(".section") and ".text." in l][0]
cur, m = None, {}
for l in sass[st + 1:]:
    if l.strip().startswith(".section") and ".text." in l:
        break
    if "//##" in l:
        mm = re.search(r'File "([^"]+)", line (\d+)', l)
        if mm:
            cur = (mm.group(1).split("/")[-1], int(mm.group(2)))
    mo = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mo and cur is not None:
        m[int(mo.group(1), 16)] = cur
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"],
                                      capture_output=True, text=True).stdout.splitlines()))
h = rows[1]
col = {n: h.index(n) for n in ("Address", "L2 Theoretical Sectors Global",
                              "L2 Theoretical Sectors Global Excessive",
                              "Warp Stall Sampling (All Samples)", "Instructions Executed")}
base = int(rows[2][col["Address"]], 16)
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
for r in rows[2:]:
    a = agg[m.get(int(r[col["Address"]], 16) - base, ("?", 0))]
    for k, c in enumerate(("L2 Theoretical Sectors Global", "L2 Theoretical Sectors Global Excessive",
                           "Warp Stall Sampling (All Samples)", "Instructions Executed")):
        a[k] += int(float(r[col[c]] or 0))
W = sum(a[2] for a in agg.values()) or 1
src = {}
for key, a in sorted(agg.items(), key=lambda x: -x[1][2])[:top]:
    f, ln = key
    if f not in src:
        try:
            src[f] = open("paper_2309_15676_b200/csrc/" + f).read().splitlines()
        except OSError:
            src[f] = []
    text = src[f][ln - 1].strip()[:70] if 0 < ln <= len(src[f]) else ""
    print(f"{f}:{ln} stall={a[2] / W:.1%} inst={a[3]} sect={a[0]} exc={a[1]} | {text}")
