"""Throughput view of one dataflow acceptance (RCB_PROFILE=1), any size:
fetch / decide rates over the span, decide-latency percentiles split by
decision path (box-simple or not), and the box-wait share.

  python tools/df_rate.py ITERATION CONFIG
"""
import ctypes as C
import os
import sys

os.environ["RCB_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402

it_target = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sc = scenes.CONFIGS[sys.argv[2]]() if len(sys.argv) > 2 else scenes.cfg4()
eng = P.RegionCompetition(sc.image, sc.labels,
                          P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                          P.SobolevParams(sc.length_scale),
                          P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace,
                                            drift_tolerance=1e-3))
for _ in range(it_target):
    eng.iterate()
cap = eng.last_negative + 1
n = C.c_int64()
t = np.zeros(4 * cap, np.int64)
P._lib.check(P._lib.lib.rcb_engine_debug_times(eng._h, P._lib.ptr(t), cap, C.byref(n)))
part = np.zeros(cap, np.int32)
code = np.zeros(cap, np.int32)
P._lib.check(P._lib.lib.rcb_engine_debug_codes(eng._h, P._lib.ptr(part), P._lib.ptr(code), cap,
                                               C.byref(n)))
m = n.value
t = t[:4 * m].reshape(m, 4).astype(np.float64)
t0 = t[:, 0].min()
f, d, tb, tw = ((t[:, k] - t0) / 1e3 for k in range(4))
code = code[:m]
span = d.max()
print(f"iteration {it_target}: {m} candidates, span {span:.0f} us, "
      f"{m / span:.1f} decisions/us, counters {eng.counters()}")
for q in (0.1, 0.5, 0.9, 0.99, 1.0):
    print(f"  fetched by q{q}: {np.quantile(f, q):9.1f} us   decided by q{q}: {np.quantile(d, q):9.1f} us")
lat = d - f
boxw = tb - f
simple = code == 0
for name, sel in (("box-simple", simple), ("other", ~simple)):
    if sel.any():
        print(f"  {name:10s} n {int(sel.sum()):9d}  latency us p50 {np.median(lat[sel]):7.1f} "
              f"p90 {np.percentile(lat[sel], 90):7.1f} p99 {np.percentile(lat[sel], 99):8.1f}  "
              f"box-wait p50 {np.median(boxw[sel]):7.1f} p90 {np.percentile(boxw[sel], 90):7.1f}")
# warp-time budget: sum of latencies vs warps x span
print(f"  sum of per-candidate latencies {lat.sum() / 1e6:.2f} s "
      f"(warp-seconds; box waits {boxw.sum() / 1e6:.2f} s)")
