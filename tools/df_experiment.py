"""Timing experiments on one dataflow acceptance: run a config to iteration
N-1, snapshot nothing, then time iteration N under each environment setting
given on the command line (each on a fresh engine, since an experiment such
as RCB_DF_NOWAIT=1 produces wrong labels).

  python tools/df_experiment.py cfg4 20 "" RCB_DF_NOWAIT=1 RCB_DF_CLAIM=chunk
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402

cfg, it_target = sys.argv[1], int(sys.argv[2])
sc = scenes.CONFIGS[cfg]()
for setting in sys.argv[3:]:
    eng = P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                              P.SobolevParams(sc.length_scale),
                              P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3))
    for _ in range(it_target - 1):
        eng.iterate()
    kv = [s.split("=", 1) for s in setting.split(",") if s]
    for k, v in kv:
        os.environ[k] = v
    try:
        rec = eng.iterate()
        t = [round(x, 2) for x in eng.timings()[0]]
        print(f"[{setting}] moves {rec.moves} timings {t}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"[{setting}] failed: {e}", flush=True)
    for k, _ in kv:
        os.environ.pop(k, None)
    del eng
