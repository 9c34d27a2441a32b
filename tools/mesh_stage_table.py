"""Per-stage table of one configs[4] iteration from the ncu launch list that
tools/profile_mesh.sh writes (gpurun_out/pm_launches.csv): time share, DRAM
bytes and GB/s, issue activity and SIMT lanes per stage (last iteration)."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/pm_launches.csv"
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    d = L.setdefault(r[h.index("ID")], {"k": r[h.index("Kernel Name")]})
    d[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
launches = list(L.values())
gen = [i for i, x in enumerate(launches) if "wf_gen" in x["k"]]
while gen[-1] >= 1 and "tex_ilv" in launches[gen[-1] - 1]["k"]:
    gen[-1] -= 1
last = launches[gen[-1]:]


def stage(name):
    for s in ("tex_ilv", "wf_gen", "wf_isect", "wf_shade", "wf_shadow", "wf_tail", "wf_scatter",
              "finalize", "meta_update_fixed", "meta_update"):
        if s in name:
            return s
    return name.split("(")[0][-30:]


agg = collections.OrderedDict()
for x in last:
    a = agg.setdefault(stage(x["k"]), collections.Counter())
    t = x["gpu__time_duration.sum"]
    a["n"] += 1
    a["ns"] += t
    a["bytes"] += x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"]
    a["issue_w"] += x["smsp__issue_active.avg.pct_of_peak_sustained_active"] * t
    a["lanes_w"] += x["smsp__thread_inst_executed_per_inst_executed.ratio"] * t
    a["warps_w"] += x["sm__warps_active.avg.pct_of_peak_sustained_active"] * t
tot = sum(a["ns"] for a in agg.values())
print("| stage | launches | us | share | DRAM MB | DRAM GB/s | issue active % | lanes/warp-inst | warps active % |")
print("|---|---|---|---|---|---|---|---|---|")
for k, a in agg.items():
    print(f"| {k} | {a['n']} | {a['ns']/1e3:.0f} | {a['ns']/tot:.3f} | {a['bytes']/1e6:.0f} | "
          f"{a['bytes']/a['ns']:.0f} | {a['issue_w']/a['ns']:.1f} | {a['lanes_w']/a['ns']:.1f} | "
          f"{a['warps_w']/a['ns']:.1f} |")
print(f"| total | {sum(a['n'] for a in agg.values())} | {tot/1e3:.0f} | 1 | "
      f"{sum(a['bytes'] for a in agg.values())/1e6:.0f} | | | | |")
