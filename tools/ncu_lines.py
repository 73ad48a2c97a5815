"""Top source lines by warp-stall samples from an ncu report (source page).

  python tools/ncu_lines.py report.ncu-rep [function-substring] [n]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall") and "Not Issued" not in h]


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


src = []
for r in rows:
    if len(r) > 5 and r[0] not in ("", "Line No") and r[0].isdigit():
        src.append((num(r[4]), int(r[0]), r[1].strip()[:80],
                    sorted(((hdr[i][6:], num(r[i])) for i in cols), key=lambda x: -x[1])[:3]))
tot = sum(x[0] for x in src)
print("samples", tot)
for s, ln, t, top in sorted(src, key=lambda x: -x[0])[:n]:
    print(f"{s:7d} {100 * s / max(tot, 1):5.1f}% L{ln}: {t:80s} {top}")
