"""Aggregate RCB_PROFILE stage timers and iterate() phases over a config run.

  RCB_PROFILE=1 python tools/config_run.py --config cfg2 > prof.txt 2>&1
  python tools/stage_profile.py prof.txt
"""
import collections
import json
import re
import sys

st = collections.defaultdict(float)
ph = [0.0] * 5
rows = 0
tot = 0.0
for line in open(sys.argv[1]):
    m = re.match(r"\[rcb\] (\S+)\s+([\d.]+) ms", line)
    if m:
        st[m.group(1)] += float(m.group(2))
        continue
    if line.startswith('{"it"'):
        d = json.loads(line)
        rows += 1
        tot += d["ms"]
        ph = [a + b for a, b in zip(ph, d["phases"])]
print("iterations", rows, "device ms", round(tot, 1))
print("phases ms (extract, energy, sobolev, rank, accept):", [round(x, 1) for x in ph])
print("accept stages ms:", {k: round(v, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])})
