"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
python scripts/launch_summary.py launches.csv [top]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hdr]
ki, vi, gi, bi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size'), h.index('Block Size')
mi = h.index('Metric Name') if 'Metric Name' in h else None
tot = 0.0
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) < len(h) or (mi is not None and r[mi] != 'gpu__time_duration.sum'):
        continue
    t = float(r[vi].replace(',', '')) / 1e3
    tot += t
    k = r[ki].split('(')[0][:44] + ' grid' + r[gi] + ' blk' + r[bi]
    agg.setdefault(k, []).append(t)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:top]:
    print('%9.1f us  n=%4d  avg %8.1f  %s' % (sum(v), len(v), sum(v) / len(v), k))
print('total us', round(tot, 1), 'launches', sum(len(v) for v in agg.values()))
