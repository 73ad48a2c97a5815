"""Per-rank device time of the z-slab sharded iteration, measured on ONE GPU.

G slab engines of the same volume run in lock step (shard.LocalSlabGroup: all
score, the slabs' scores are copied into place, all finish, the band-ledger
limbs are summed; no kernel waits on another engine), so each engine's event
timers see what its rank would execute on its own GPU.  The iteration time of
a G-GPU run is modelled as the slowest rank's device time, median over the
window (the all-gather of the scores and the 68-limb all-reduce over NVLink
are not included).

  python tools/slab_model.py [--n 512] [--warm 5] [--iters 10] [--ranks 1,2,4,8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402
from paper_1403_0240_b200.shard import LocalSlabGroup  # noqa: E402


def make(sc):
    return P.RegionCompetition(sc.image, sc.labels,
                               P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                               P.SobolevParams(sc.length_scale),
                               P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace,
                                                 drift_tolerance=1e-3))


def lockstep(group):
    """LocalSlabGroup.iterate with a device synchronisation after every
    engine's turn, so no two engines' kernels overlap on the one GPU and each
    engine's event timers see its own work only."""
    import torch
    t0 = [e._pre_iterate() for e in group.engines]
    infos = []
    for s in group.slabs:
        infos.append(s.score())
        torch.cuda.synchronize()
    ranges = group.slabs[0].ranges()
    bufs = [s.buffers(i, e.device) for s, i, e in zip(group.slabs, infos, group.engines)]
    for r, (a, b) in enumerate(ranges):
        for j in range(len(group.engines)):
            if j != r and b > a:
                for dst, src in zip(bufs[j], bufs[r]):
                    dst[a:b].copy_(src[a:b])
    torch.cuda.synchronize()
    recs = []
    for s in group.slabs:
        recs.append(s.finish())
        torch.cuda.synchronize()
    limbs = [s.band_limbs(e.device)[0] for s, e in zip(group.slabs, group.engines)]
    if any(l is not None for l in limbs):
        total = sum(l.clone() for l in limbs)
        for l in limbs:
            l.copy_(total)
        torch.cuda.synchronize()
        recs = [s.band_apply(r) for s, r in zip(group.slabs, recs)]
    return [e._post_iterate(r, t) for e, r, t in zip(group.engines, recs, t0)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--warm", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--ranks", default="1,2,4,8")
    a = ap.parse_args()
    sc = scenes.cfg4() if a.n == 512 else scenes.cfg4(n=a.n, n_obj=max(1, 64 * a.n ** 3 // 512 ** 3),
                                                      per_axis=max(1, 8 * a.n // 512))
    base = None
    rank_ms = 0.0
    for g in [int(x) for x in a.ranks.split(",")]:
        try:
            group = LocalSlabGroup([make(sc) for _ in range(g)])
            per_rank = np.zeros((a.iters, g, 6))
            for it in range(a.warm + a.iters):
                lockstep(group)
                if it >= a.warm:
                    for r, e in enumerate(group.engines):
                        per_rank[it - a.warm, r] = e.timings()[0]
            # ev3 -> ev4 (rank order) spans the other engines' turns: take the
            # replicated rank phase from the single engine
            if g == 1:
                rank_ms = float(per_rank[:, 0, 3].mean())
            per_rank[:, :, 3] = rank_ms
            per_rank[:, :, 5] = per_rank[:, :, :5].sum(axis=2)
            # medians over the window's iterations: buffer growth in a process that
            # holds several 512^3 engines stalls single iterations by 10-400 ms
            slowest = float(np.median(per_rank[:, :, 5].max(axis=1)))
            mean_ph = np.median(per_rank.mean(axis=1), axis=0)
            if base is None:
                base = slowest
            print(json.dumps({"ranks": g, "median_ms_per_iteration_slowest_rank": round(float(slowest), 2),
                              "speedup_vs_1": round(float(base / slowest), 3),
                              "median_phase_ms_mean_over_ranks": {k: round(float(v), 2) for k, v in zip(
                                  ("extract", "energy", "sobolev", "rank", "accept+band", "iterate"), mean_ph)},
                              "window": [a.warm + 1, a.warm + a.iters], "lattice": list(sc.image.shape)}),
                  flush=True)
            del group
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"ranks": g, "error": str(ex)[:200]}), flush=True)


if __name__ == "__main__":
    main()
