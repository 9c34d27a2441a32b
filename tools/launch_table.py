"""Print the last N launches of an ncu --csv launch list (metrics per row)."""
import csv, collections, sys
path = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
data = collections.defaultdict(dict); names = {}
for r in rows[hi + 1:]:
    data[r[ii]][r[mi]] = r[vi]; names[r[ii]] = r[ki]
ids = sorted(data, key=int)
keys = sorted({k for d in data.values() for k in d})
short = {k: k.split('.')[0].replace('smsp__', '').replace('sm__', '')[:18] for k in keys}
print('kernel'.ljust(48), ' '.join(short[k].rjust(18) for k in keys))
tot = 0.0
for i in ids[-N:]:
    d = data[i]
    tot += float(d.get('gpu__time_duration.sum', 0))
    nm = names[i].split('(')[0].replace('void ', '').replace('mesh::<unnamed>::', '').replace('<unnamed>::', '')
    print(nm[:48].ljust(48), ' '.join(d.get(k, '').rjust(18) for k in keys))
print('sum of durations (ns)', tot)
