"""Where batched small images lose time: K threads each run one cfg5 image;
per image the sum of device ms (engine events) and the wall time."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
scs = [scenes.cfg5_image(i) for i in range(K)]
sc = scs[0]
ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
ocfg = P.OptimizerConfig("sobolev", max_iterations=50)
# warm-up engine (module load, pool priming)
P.RegionCompetition(scs[0].image, scs[0].labels, ecfg, P.SobolevParams(sc.length_scale), ocfg).iterate()
res = [None] * K


def work(i):
    t0 = time.time()
    eng = P.RegionCompetition(scs[i].image, scs[i].labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
    t1 = time.time()
    dev = [0.0, 0.0]

    def cb(e, r):
        t = e.timings()[0]
        dev[0] += t[5]
        dev[1] += t[4]
    eng.run(on_iteration=cb)
    res[i] = {"create_s": round(t1 - t0, 3), "run_wall_s": round(time.time() - t1, 3),
              "device_s": round(dev[0] / 1e3, 3), "accept_s": round(dev[1] / 1e3, 3)}


t0 = time.time()
th = [threading.Thread(target=work, args=(i,)) for i in range(K)]
[t.start() for t in th]
[t.join() for t in th]
print(json.dumps({"threads": K, "wall_s": round(time.time() - t0, 3), "per_image": res}))
