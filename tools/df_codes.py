"""Decision-path census of one dataflow acceptance: how many candidates each
path (local box, window verdicts, BFS tiers, deferred assist jobs) decided,
and how many of those were accepted.

  python tools/df_codes.py ITERATION CONFIG
"""
import ctypes as C
import os
import sys
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402

it_target = int(sys.argv[1]) if len(sys.argv) > 1 else 40
sc = scenes.CONFIGS[sys.argv[2]]() if len(sys.argv) > 2 else scenes.cfg3()
eng = P.RegionCompetition(sc.image, sc.labels,
                          P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                          P.SobolevParams(sc.length_scale),
                          P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace,
                                            drift_tolerance=1e-3))
for _ in range(it_target):
    rec = eng.iterate()
xs, ow, cm, rk = eng.last_candidates
cap = len(xs) + 1
n = C.c_int64()
part = np.zeros(cap, np.int32)
code = np.zeros(cap, np.int32)
P._lib.check(P._lib.lib.rcb_engine_debug_codes(eng._h, P._lib.ptr(part), P._lib.ptr(code), cap,
                                               C.byref(n)))
m = n.value
part, code = part[:m], code[:m]
acc = eng.last_accepted
accset = set(zip(acc[:, 0].tolist(), acc[:, 2].tolist()))
ok = np.array([(int(xs[p]), int(cm[p])) in accset for p in part])


def path(c):
    if c == 0:
        return "box"
    job = c >= 1000000000
    c2 = c % 1000000000
    box = c2 >= 100000000
    c2 %= 100000000
    w31 = c2 // 10000000
    c2 %= 10000000
    w63 = c2 // 1000000
    c2 %= 1000000
    lev = c2 // 10000
    wb = (c2 // 100) % 10 - 2
    r = (c2 % 100) // 10 - 1
    if r < 0:
        return f"window={wb}"
    lvl = "lv<10" if lev < 10 else "lv<50" if lev < 50 else "lv>=50"
    return f"{'job' if job else 'bfs'}{'-box' if box else '-hash'} r={r} {lvl}"


cnt = Counter()
acc_c = Counter()
for c, a in zip(code.tolist(), ok.tolist()):
    k = path(c)
    cnt[k] += 1
    acc_c[k] += int(a)
print(f"iteration {rec.iteration}: {m} candidates, {len(acc)} moves, counters {eng.counters()}")
for k, v in sorted(cnt.items(), key=lambda kv: -kv[1]):
    print(f"{k:28s} {v:7d}  accepted {acc_c[k]:7d}")

# deferred assist jobs: duration (low-water reached -> answered) and the gap
# between one job's answer and the next job's start (RCB_PROFILE=1 only)
if os.environ.get("RCB_PROFILE") == "1":
    t = np.zeros(4 * cap, np.int64)
    P._lib.check(P._lib.lib.rcb_engine_debug_times(eng._h, P._lib.ptr(t), cap, C.byref(n)))
    t = t[:4 * m].reshape(m, 4)
    job = code >= 1000000000
    js, je = t[job, 2], t[job, 3]
    o = np.argsort(js)
    js, je = js[o], je[o]
    dur = (je - js) / 1e3
    gap = (js[1:] - je[:-1]) / 1e3
    span = (t[:, 1].max() - t[:, 0].min()) / 1e3
    print(f"jobs {len(js)}: duration us p50 {np.median(dur):.1f} p90 {np.percentile(dur, 90):.1f} "
          f"sum {dur.sum():.0f}; gap us p50 {np.median(gap):.1f} p90 {np.percentile(gap, 90):.1f} "
          f"sum {gap.sum():.0f}; acceptance span {span:.0f} us")
    ready = t[job, 0][o]
    print(f"  per job: scan/rebuild us p50 {np.median((ready - js) / 1e3):.1f} "
          f"p90 {np.percentile((ready - js) / 1e3, 90):.1f}; query+verdict us p50 "
          f"{np.median((je - ready) / 1e3):.1f} p90 {np.percentile((je - ready) / 1e3, 90):.1f}")
