"""Where the dataflow acceptance's warp time goes (RCB_PROFILE=1 stamps): per
candidate fetch -> box settled -> window done -> decided, summed by decision
path.

  python tools/df_phases.py 20 cfg4
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
eng = P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                          P.SobolevParams(sc.length_scale),
                          P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3))
for _ in range(it_target - 1):
    eng.iterate()
eng.iterate()
n = C.c_int64()
cap = int(os.environ.get("DF_CAP", "40000000"))
t = np.zeros(4 * cap, np.int64)
part = np.zeros(cap, np.int32)
code = np.zeros(cap, np.int32)
P._lib.check(P._lib.lib.rcb_engine_debug_times(eng._h, P._lib.ptr(t), cap, C.byref(n)))
P._lib.check(P._lib.lib.rcb_engine_debug_codes(eng._h, P._lib.ptr(part), P._lib.ptr(code), cap, C.byref(n)))
m = n.value
f, d, tb, tw = (t[k:4 * m:4].astype(np.float64) for k in range(4))
t0 = f.min()
f, d, tb, tw = ((u - t0) / 1e3 for u in (f, d, tb, tw))
code = code[:m]
span = d.max()
print("candidates", m, "span us", round(span, 1), "decisions/us", round(m / span, 1))
simple = code == 0
win = (code >= 1000) & ((code // 10) % 10 == 0)
bfs = (code >= 1000) & ((code // 10) % 10 > 0)
w5 = win & (code % 10 == 7)
for name, sel in (("all", np.ones(m, bool)), ("simple", simple), ("window", win), ("  of which 5^3", w5), ("bfs", bfs)):
    k = int(sel.sum())
    if not k:
        continue
    box, wn, bf = (tb - f)[sel], (tw - tb)[sel], (d - tw)[sel]
    print(f"{name:14s} n {k:9d}  warp-us total: box {box.sum() / 1e3:9.1f} ms  win {wn.sum() / 1e3:9.1f} ms  rest {bf.sum() / 1e3:9.1f} ms"
          f" | box p50 {np.percentile(box, 50):6.2f} p90 {np.percentile(box, 90):7.2f} p99 {np.percentile(box, 99):8.2f} mean {box.mean():7.2f}"
          f" | win mean {wn.mean():7.2f} rest mean {bf.mean():8.2f}")
lat = d - f
print("total warp-ms fetch->decided", round(lat.sum() / 1e3, 1), " per-warp (2368 warps) ms", round(lat.sum() / 1e3 / 2368, 2))
# fetch gaps: time between consecutive fetches (claim order) ~ throughput over time
order = np.argsort(f)
print("box histogram us [0,.5,1,1.5,2,3,5,10,20,50,100,1e9):",
      np.histogram(tb - f, bins=[0, .5, 1, 1.5, 2, 3, 5, 10, 20, 50, 100, 1e9])[0].tolist())
# stragglers: long topology tests and when the kernel would end without them
rest = d - tw
for thr in (500, 1000, 2000, 5000, 10000):
    sel = rest > thr
    print(f"candidates with > {thr} us after the window test: {int(sel.sum())}, warp-ms {rest[sel].sum() / 1e3:.1f}")
nolong = d[rest <= 1000]
print("last decision among candidates without a long test: %.1f us; kernel span %.1f us" % (nolong.max(), span))
dd = np.sort(d)
for q in (0.99, 0.999, 0.9999):
    print(f"decided by {q}: {dd[int(q * (m - 1))]:.1f} us")
