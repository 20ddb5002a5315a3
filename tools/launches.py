#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum CSV) by kernel+grid."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
gi = h.index('Grid Size') if 'Grid Size' in h else None
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(',', ''))
    v *= {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6}.get(r[ui], 1)
    name = r[ki].split('(')[0].replace('hs::', '').replace('<unnamed>::', '')
    k = name + (' grid=' + r[gi] if gi is not None else '')
    agg[k][0] += 1
    agg[k][1] += v
    seq.append((k, v))
tot = sum(v[1] for v in agg.values())
print(f"{len(seq)} launches, {tot / 1e6:.2f} ms total")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{v[0]:6d} {v[1] / 1e6:9.3f}ms {v[1] / v[0] / 1e3:9.2f}us {100 * v[1] / tot:5.1f}%  {k}")
