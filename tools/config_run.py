"""Run a BASELINE config on one GPU through the public API and print the
per-iteration trace (device ms, moves, particles, ledger) as JSON lines.

  python tools/config_run.py --config cfg3 --iters 100
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--drift", type=float, default=1e-3)
    a = ap.parse_args()
    t0 = time.time()
    sc = scenes.CONFIGS[a.config]()
    t_gen = time.time() - t0
    iters = a.iters or sc.iterations
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=a.drift,
                             max_iterations=iters)
    t0 = time.time()
    eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
    t_init = time.time() - t0
    print(json.dumps({"config": a.config, "shape": list(sc.image.shape), "labels": int(sc.labels.max()),
                      "gen_s": round(t_gen, 2), "engine_init_s": round(t_init, 3)}), flush=True)
    tot = 0.0
    t_wall = time.time()

    def cb(e, rec):
        nonlocal tot
        t, nl = e.timings()
        c = e.counters()
        tot += t[5]
        print(json.dumps({"it": rec.iteration, "ms": round(t[5], 3), "host_s": round(rec.seconds, 4),
                          "moves": rec.moves, "particles": rec.particles, "energy": rec.energy,
                          "mode": rec.mode, "negative": c["negative"], "pairs": e.last_pairs,
                          "bfs": c["bfs_runs"], "deferred": c["deferred"],
                          "phases": [round(x, 3) for x in t[:5]]}), flush=True)

    res = eng.run(on_iteration=cb)
    wall = time.time() - t_wall
    print(json.dumps({"status": res.status, "iterations": res.iterations,
                      "final_energy": res.final_energy.total, "regions": res.region_count,
                      "device_ms_total": round(tot, 2), "wall_s": round(wall, 3),
                      "iterations_per_s_wall": res.iterations / wall}), flush=True)


if __name__ == "__main__":
    main()
