"""Per-kernel DRAM bytes and durations from an ncu report (raw page) into
profiles/r01_traffic.json, whose energy_plus_sobolev_dram_bytes bench.py
reports as roofline.traffic.

  python tools/ncu_traffic.py report.ncu-rep "source description" [out.json]
"""
import csv
import json
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics",
                      "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
ix = {k: i for i, k in enumerate(h)}
scale = {"Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3,
         "msecond": 1e3, "ms": 1e3, "us": 1, "ns": 1e-3}


def val(r, k):
    return float(r[ix[k]].replace(",", "")) * scale.get(units[ix[k]], 1)


kern = {}
for r in rows[2:]:
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("rcb::", "")
    kern[name] = {"dram_bytes": int(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")),
                  "us": round(val(r, "gpu__time_duration.sum"), 3)}
e = sum(v["dram_bytes"] for k, v in kern.items()
        if k.startswith(("k_delta_ps", "k_sobolev", "k_sob_pack")))
doc = {"source": sys.argv[2], "kernels": kern, "energy_plus_sobolev_dram_bytes": e}
with open(sys.argv[3] if len(sys.argv) > 3 else "profiles/r01_traffic.json", "w") as fh:
    json.dump(doc, fh, indent=1)
print(json.dumps(doc, indent=1))
