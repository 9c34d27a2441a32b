"""Print an ncu --csv launch log as one row per launch (kernel, metrics)."""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    out = {}
    for r in rows[hi + 1:]:
        d = out.setdefault(r[h.index("ID")], {"k": r[h.index("Kernel Name")].split("(")[0][-40:]})
        d[r[h.index("Metric Name")].split(".")[0][-28:]] = r[h.index("Metric Value")]
    for i, d in out.items():
        print(path.split("/")[-1], i, "  ".join(f"{k}={v}" for k, v in d.items()))
