"""Per-iterate device time on cfg2 under different conditions: after an L2
flush (bench default), without the flush, and back-to-back (queue kept full)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402

sc = scenes.cfg2()
mk = lambda: P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig("ps", "poisson", smooth_radius=4),
                                 P.SobolevParams(6.0), P.OptimizerConfig("sobolev", vanish_grace=5,
                                                                        drift_tolerance=1e-3))
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for mode in ("flush", "flush+idle", "noflush", "backtoback"):
    eng = mk()
    st = torch.cuda.ExternalStream(eng.stream)
    for _ in range(5):
        eng.iterate()
    torch.cuda.synchronize()
    tot = 0.0
    steps = []
    wall = time.perf_counter()
    if mode == "backtoback":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            eng.iterate()
        e1.record(st)
        e1.synchronize()
        tot = e0.elapsed_time(e1)
    else:
        for _ in range(20):
            if mode.startswith("flush"):
                flush.zero_()
            if mode == "flush+idle":
                torch.cuda.synchronize()
                time.sleep(0.1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            eng.iterate()
            e1.record(st)
            e1.synchronize()
            steps.append(round(e0.elapsed_time(e1), 2))
            tot += e0.elapsed_time(e1)
    wall = time.perf_counter() - wall - (2.0 if mode == "flush+idle" else 0.0)
    t, nl = eng.timings()
    print(f"{mode:10s} device ms/iter {tot / 20:.3f}  wall ms/iter {1e3 * wall / 20:.3f}  "
          f"(engine phases last: {[round(x, 3) for x in t]})", steps, flush=True)
