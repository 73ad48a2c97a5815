"""Critical-path view of one dataflow acceptance (RCB_PROFILE=1): per rank
position, when its warp fetched it and when it was decided."""
import ctypes as C
import os
import sys

os.environ["RCB_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402

it_target = int(sys.argv[1]) if len(sys.argv) > 1 else 19
sc = scenes.cfg2()
eng = P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig("ps", "poisson", smooth_radius=4),
                          P.SobolevParams(6.0), P.OptimizerConfig("sobolev", vanish_grace=5, drift_tolerance=1e-3))
for _ in range(it_target):
    eng.iterate()
n = C.c_int64()
cap = 400000
t = np.zeros(2 * cap, np.int64)
part = np.zeros(cap, np.int32)
code = np.zeros(cap, np.int32)
P._lib.check(P._lib.lib.rcb_engine_debug_times(eng._h, P._lib.ptr(t), cap, C.byref(n)))
P._lib.check(P._lib.lib.rcb_engine_debug_codes(eng._h, P._lib.ptr(part), P._lib.ptr(code), cap, C.byref(n)))
m = n.value
f, d = t[0:2 * m:2], t[1:2 * m:2]
t0 = f.min()
f = (f - t0) / 1e3
d = (d - t0) / 1e3
print("candidates", m, "span us", d.max(), "counters", eng.counters())
lat = d - f
print("decide-latency us: p50 %.1f p90 %.1f p99 %.1f max %.1f" % tuple(np.percentile(lat, [50, 90, 99, 100])))
print("fetch time us: p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(f, [50, 90, 100])))
for q in (0.5, 0.9, 0.99, 0.999, 1.0):
    print(f"decided by {q:6.3f} of candidates: {np.quantile(d, q):9.1f} us")
slow = np.argsort(-lat)[:15]
print("slowest (pos, code, fetch, latency):")
for p in slow:
    print(int(p), int(code[p]), round(f[p], 1), round(lat[p], 1))
# how many candidates are decided after 50% of the span
