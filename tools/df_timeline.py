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
sc = scenes.CONFIGS[sys.argv[2]]() if len(sys.argv) > 2 else scenes.cfg2()
eng = P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                          P.SobolevParams(sc.length_scale),
                          P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3))
for _ in range(it_target - 1):
    eng.iterate()
cnt0 = eng.model.stats.count.copy()
eng.iterate()
n = C.c_int64()
cap = int(os.environ.get("DF_CAP", "400000"))
t = np.zeros(4 * cap, np.int64)
part = np.zeros(cap, np.int32)
code = np.zeros(cap, np.int32)
P._lib.check(P._lib.lib.rcb_engine_debug_times(eng._h, P._lib.ptr(t), cap, C.byref(n)))
P._lib.check(P._lib.lib.rcb_engine_debug_codes(eng._h, P._lib.ptr(part), P._lib.ptr(code), cap, C.byref(n)))
m = n.value
f, d, tb, tw = (t[k:4 * m:4] for k in range(4))
t0 = f.min()
f, d, tb, tw = ((u - t0) / 1e3 for u in (f, d, tb, tw))
print("candidates", m, "span us", d.max(), "counters", eng.counters())
lat = d - f
print("decide-latency us: p50 %.1f p90 %.1f p99 %.1f max %.1f" % tuple(np.percentile(lat, [50, 90, 99, 100])))
print("fetch time us: p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(f, [50, 90, 100])))
for q in (0.5, 0.9, 0.99, 0.999, 1.0):
    print(f"decided by {q:6.3f} of candidates: {np.quantile(d, q):9.1f} us")
hist, edges = np.histogram(d, bins=20)
print("decisions per 5% of the span:", hist.tolist(), "span us", round(float(d.max()), 1))
lat_hist = np.histogram(lat, bins=[0, 1, 2, 5, 10, 20, 50, 100, 200, 500, 1e9])[0]
print("latency histogram us [0,1,2,5,10,20,50,100,200,500,inf):", lat_hist.tolist())
slow = np.argsort(-lat)[:15]
print("slowest (pos, code, fetch, latency):")
for p in slow:
    print(int(p), int(code[p]), round(f[p], 1), round(lat[p], 1))
# how many candidates are decided after 50% of the span
defer = code >= 1000000000
code = code % 1000000000
boxt = code >= 100000000
print('box-tier candidates', int(boxt.sum()), 'deferred', int(defer.sum()))
code = code % 100000000
w31 = code // 10000000 - 1
print('window31 runs', int((w31 >= 0).sum()), 'verdicts 1/2/0:', int((w31 == 1).sum()), int((w31 == 2).sum()), int((w31 == 0).sum()))
code = code % 10000000
w63 = code // 1000000 - 1
print('window63 runs', int((w63 >= 0).sum()), 'verdicts 1/2/0:', int((w63 == 1).sum()), int((w63 == 2).sum()), int((w63 == 0).sum()))
code = code % 1000000
lv = code // 10000
bfs = lv > 0
print("BFS candidates", int(bfs.sum()), "levels p50/p90/p99/max", np.percentile(lv[bfs], [50, 90, 99, 100]) if bfs.any() else None)
big = np.argsort(-lat)[:8]
print("slowest: levels", [int(lv[p]) for p in big], "latency", [round(float(lat[p]), 1) for p in big])
print("slowest phases (box wait, window wait, bfs):")
for p in np.argsort(-lat)[:12]:
    print("  pos", int(p), "box %.1f win %.1f bfs %.1f" % (tb[p] - f[p], tw[p] - tb[p], d[p] - tw[p]), "code", int(code[p]))
late = np.argsort(-d)[:200]
print("latest 200 mean phases: box %.1f win %.1f bfs %.1f" % ((tb - f)[late].mean(), (tw - tb)[late].mean(), (d - tw)[late].mean()))

xs, ow, cm, rk = eng.last_candidates
neg = rk < 0
nown = np.bincount(ow[neg], minlength=len(cnt0))
small = (np.arange(len(cnt0)) > 0) & (cnt0 - nown[:len(cnt0)] <= 1)
pa, pb = ow[part[:m]], cm[part[:m]]
inv = small[pa] | small[pb]
print("small labels", int(small.sum()), "candidates involving them", int(inv.sum()))
slow = np.argsort(-lat)[:40]
print("slowest 40: involve small label:", int(inv[slow].sum()), " owner small:", int(small[pa][slow].sum()))
late = d > np.quantile(d, 0.99)
print("last 1%: involve small label", int(inv[late].sum()), "of", int(late.sum()))

# inherent dependency depth: position p waits on every earlier position whose
# pixel lies in p's 3x3 box (the minimum read set of the simple-point test)
W = sc.image.shape[-1]
px = xs[part[:m]]
best = {}
depth = np.zeros(m, np.int32)
for p in range(m):
    x = int(px[p]); r, c = divmod(x, W)
    dmax = 0
    for dr in (-1, 0, 1):
        for dc in (-1, 0, 1):
            v = best.get((r + dr) * W + c + dc, 0)
            if v > dmax:
                dmax = v
    depth[p] = dmax + 1
    if depth[p] > best.get(x, 0):
        best[x] = depth[p]
print("box-dependency critical path", int(depth.max()), "p99", np.percentile(depth, 99))
for q in (0.5, 0.9, 0.99, 1.0):
    sel = d >= np.quantile(d, q) - 1e-9
    print(f"decided at >= q{q}: mean depth {depth[sel].mean():.1f}")
late = np.argsort(-d)[:10]
print("latest decided: depth", [int(depth[p]) for p in late], "time", [round(float(d[p]), 1) for p in late])
cc = np.corrcoef(depth, d)[0, 1]
print("corr(depth, decide time)", round(float(cc), 3), " us per depth level", round(float(d.max() / depth.max()), 2))

for p in np.nonzero(defer)[0]:
    print("deferred pos %d fetch %.1f lowmark %.1f job %.1f decided %.1f (job us %.1f)" %
          (p, f[p], tb[p], tw[p], d[p], tw[p] - tb[p]))
bt = d - tw
code = code[:m]
retries = code % 10
isb = (code // 10) % 10 > 0
lvl = code // 10000
sel0 = isb & (retries == 0) & (lvl > 0)
if sel0.any():
    per = bt[sel0] / lvl[sel0]
    print("BFS no-retry: n %d, us/level p50 %.2f p90 %.2f, bfs us p50 %.1f p90 %.1f max %.1f" %
          (sel0.sum(), np.median(per), np.percentile(per, 90), np.median(bt[sel0]),
           np.percentile(bt[sel0], 90), bt[sel0].max()))
sel1 = isb & (retries > 0)
print("BFS with retries: n %d, retries mean %.2f, bfs us p50 %.1f max %.1f" %
      (sel1.sum(), retries[sel1].mean() if sel1.any() else 0, np.median(bt[sel1]) if sel1.any() else 0,
       bt[sel1].max() if sel1.any() else 0))
how = (code % 10000) // 1000
wbv = (code % 1000) // 100 - 2
print("candidates needing the window test:", int((how == 1).sum()), "of", m,
      " window verdicts 1/2/0:", int(((how == 1) & (wbv == 1)).sum()), int(((how == 1) & (wbv == 2)).sum()),
      int(((how == 1) & (wbv == 0)).sum()))
bl = lvl[isb]
for R in (7, 10, 15, 20):
    print(f"  BFS with <= {R} levels: {int((bl <= R).sum())} of {len(bl)}")
