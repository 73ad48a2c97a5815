"""Copy the outputs of tools/gpurun/gpurun_final.sh from gpurun_out/ into profiles/ under a
round tag and write the launch-list summaries and the K5 + K6 traffic file bench.py reads.

  python tools/store_profiles.py [r02b]
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02b"
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
for src, dst in (("final_bench.json", "bench.json"), ("final_bench_ref.json", "bench_ref.json"),
                 ("final_pytest_gpu.log", "pytest_gpu.log"),
                 ("final_launches_cfg4.csv", "launches_cfg4.csv"),
                 ("final_launches_cfg2.csv", "launches_cfg2.csv"),
                 ("final_ncu_full_cfg4.csv", "ncu_full_cfg4.csv")):
    shutil.copy(os.path.join(G, src), os.path.join(P, f"{tag}_{dst}"))
tw = os.path.join(ROOT, "tools", "traffic_window.py")
l4 = os.path.join(P, f"{tag}_launches_cfg4.csv")
subprocess.run([sys.executable, tw, l4, "20", os.path.join(P, f"{tag}_traffic_cfg4.json")],
               check=True, stdout=subprocess.DEVNULL)
subprocess.run([sys.executable, tw, l4, "20", "/tmp/_all.json", "."], check=True,
               stdout=subprocess.DEVNULL)
d = json.load(open("/tmp/_all.json"))
ks = sorted(d["kernels"].items(), key=lambda kv: -kv[1]["us_per_iteration"])
tot = sum(v["us_per_iteration"] for _, v in ks)
lines = ["cfg4 iterations 6-25 (tools/profile_window.py --warm 5 --iters 20), ncu "
         "gpu__time_duration.sum + dram bytes, per iteration",
         f"total {tot / 1e3:.2f} ms per iteration over "
         f"{sum(v['launches'] for _, v in ks) / 20:.1f} launches per iteration"]
for k, v in ks[:25]:
    lines.append(f"{v['us_per_iteration']:10.1f} us {v['us_per_iteration'] / tot * 100:5.1f}% "
                 f"{v['dram_bytes_per_iteration'] / 1e9:7.2f} GB DRAM {v['launches'] / 20:5.1f} launches  {k[:80]}")
open(os.path.join(P, f"{tag}_launches_cfg4_summary.txt"), "w").write("\n".join(lines) + "\n")
out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"),
                      os.path.join(P, f"{tag}_launches_cfg2.csv"), "16"], check=True,
                     capture_output=True, text=True).stdout
open(os.path.join(P, f"{tag}_launches_cfg2_summary.txt"), "w").write(out)
b = json.load(open(os.path.join(P, f"{tag}_bench.json")))
print("\n".join(lines[:8]))
print(out.splitlines()[0])
print("bench: value %.4g ms/step %.2f e2e %.4g roofline frac %.4f traffic %s fp32 %.4g cfg2 it/s %.0f full run %.1f ms" % (
    b["value"], b["ms_per_step"], b["e2e"]["value"], b["roofline"]["frac"], b["roofline"]["traffic"],
    b["fp32_mode"]["value"], b["cfg2"]["iterations_per_s"], b["cfg2"]["full_run"]["device_ms"]))
print("w=1 sweep:", [(p["point"], round(p["hbm_frac"], 3)) for p in b["k6_sweep"] if p["width"] == 1])
print(open(os.path.join(P, f"{tag}_pytest_gpu.log")).read().strip().splitlines()[-2:])
