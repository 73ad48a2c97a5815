import sys, time, json, os
sys.path.insert(0, os.getcwd())
import paper_1403_0240_b200 as P, scenes
sc = scenes.cfg5_image(0)
ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
ocfg = P.OptimizerConfig("sobolev", max_iterations=50)
for rep in range(2):
    t0 = time.time()
    eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
    t1 = time.time()
    ms = []
    def cb(e, r):
        ms.append(e.timings()[0][5])
    res = eng.run(on_iteration=cb)
    t2 = time.time()
    print(json.dumps({"create_s": round(t1 - t0, 4), "run_s": round(t2 - t1, 4), "iters": res.iterations,
                      "device_ms_sum": round(sum(ms), 2), "status": res.status, "ms": [round(x, 2) for x in ms]}))
print(json.dumps(eng.counters()))
