"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[r[ki][:70]][0] += 1
        agg[r[ki][:70]][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v[1]/1e3:10.1f} us {100*v[1]/tot:5.1f}% {v[0]:5d}  {k}")
