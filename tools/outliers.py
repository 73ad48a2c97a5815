import re, sys, json
for fn in sys.argv[1:]:
    stages = []
    for line in open(fn):
        m = re.match(r"\[rcb\] (\S+)\s+([\d.]+) ms", line)
        if m:
            stages.append((m.group(1), float(m.group(2))))
            continue
        if line.startswith('{"it"'):
            d = json.loads(line)
            if d["ms"] > 4:
                print(fn, d["it"], d["ms"], [s for s in stages if s[1] > 0.5])
            stages = []
