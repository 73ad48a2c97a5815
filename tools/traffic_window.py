"""ncu DRAM traffic of the energy + Sobolev kernels over bench.py's timed
window, into profiles/r02_traffic_cfg4.json (bench.py's roofline.traffic).

  ncu --profile-from-start off --clock-control none --csv \
      --kernel-name regex:'k_delta_ps|k_sob_pack|k_sobolev' \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --log-file gpurun_out/traffic.csv \
      python tools/profile_window.py --config cfg4 --warm 5 --iters 20
  python tools/traffic_window.py gpurun_out/traffic.csv 20 [out.json]
"""
import collections
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3, "second": 1e6}

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, ui, vi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
iters = int(sys.argv[2])
agg = collections.defaultdict(lambda: collections.defaultdict(float))
launches = collections.Counter()
import re  # noqa: E402

# K5 + K6: the energy and Sobolev kernels of the window (argv[4]: another regex)
KEEP = re.compile(sys.argv[4] if len(sys.argv) > 4 else r"k_delta_|k_pack_sites|k_sob_pack|k_sobolev")
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("rcb::", "")
    if not KEEP.search(name):
        continue
    v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    agg[name][r[mi]] += v
    if r[mi] == "gpu__time_duration.sum":
        launches[name] += 1
kern = {k: {"launches": launches[k],
            "dram_bytes_per_iteration": (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / iters,
            "us_per_iteration": a["gpu__time_duration.sum"] / iters}
        for k, a in agg.items()}
doc = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over cfg4 iterations "
                 f"6-25 (tools/profile_window.py --warm 5 --iters {iters}), cold-cache replay",
       "kernels": kern,
       "energy_plus_sobolev_dram_bytes_per_iteration":
           sum(v["dram_bytes_per_iteration"] for v in kern.values())}
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/r02b_traffic_cfg4.json"
with open(out, "w") as fh:
    json.dump(doc, fh, indent=1)
print(json.dumps(doc, indent=1))
