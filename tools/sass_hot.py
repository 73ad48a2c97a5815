"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kern = None
tables = []
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "Kernel Name":
        kern = r[1]
    if r and r[0] == "Address":
        h = r
        j = i + 1
        data = []
        while j < len(rows) and rows[j] and rows[j][0] not in ("Kernel Name", "Address"):
            data.append(rows[j])
            j += 1
        tables.append((kern, h, data))
        i = j
        continue
    i += 1
for kern, h, data in tables:
    si = h.index("Warp Stall Sampling (All Samples)")
    ii = h.index("Instructions Executed")
    src = h.index("Source")
    f = lambda x: float(x.replace(",", "") or 0)
    tot = sum(f(r[si]) for r in data if len(r) > si)
    print(f"== {kern[:80]}  samples={tot:.0f}  instr={sum(f(r[ii]) for r in data if len(r) > ii):.0f}")
    for r in sorted(data, key=lambda r: -f(r[si]))[:n]:
        print(f"{100 * f(r[si]) / max(tot, 1):5.1f}%  {r[0]}  {r[src][:100]}")
