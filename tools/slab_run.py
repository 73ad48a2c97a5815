"""One lattice sharded by z-slabs over the GPUs of a node (strong scaling;
DESIGN.md §9), launched like bench.py:

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
      --master-addr 127.0.0.1 --master-port 29511 tools/slab_run.py --config cfg4 \
      --warmup 5 --steps 20

One process per GPU (NCCL).  Every rank scores its slab (K1 emit, K5/K3, K6),
the slabs' scores are all-gathered in place, every rank runs the rank order
and the exact acceptance (replicated), refreshes the own-label fields of its
slab plus halo, and the band-ledger limbs are all-reduced.  Timed like
bench.py: W warm-up iterations, K iterations bracketed by a barrier and a
device synchronisation, device time by CUDA events, max over ranks; rank 0
prints one JSON line.  With one process it runs the plain engine.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402
from paper_1403_0240_b200.shard import slab_engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc = scenes.CONFIGS[a.config]()
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3)
    sob = P.SobolevParams(sc.length_scale)
    if world > 1:
        eng = slab_engine(sc.image, sc.labels, ecfg, sob, ocfg, device=local)
    else:
        eng = P.RegionCompetition(sc.image, sc.labels, ecfg, sob, ocfg, device=local)
    for _ in range(a.warmup):
        eng.iterate()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.ExternalStream(eng.stream)
    t0.record(stream)
    pairs = 0
    last = None
    for _ in range(a.steps):
        last = eng.iterate()
        pairs += eng.last_pairs  # this rank's slab of the interactions
    t1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([t0.elapsed_time(t1)], device="cuda")
    pr = torch.tensor([float(pairs)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(pr, op=dist.ReduceOp.SUM)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"config": a.config, "n_gpus": world, "scaling": "strong",
                          "steps": a.steps, "warmup": a.warmup,
                          "ms_per_step": ms.item() / a.steps,
                          "particle_interactions_per_s": pr.item() / (ms.item() / 1e3),
                          "iterations_per_s": a.steps / (ms.item() / 1e3),
                          "energy": last.energy, "moves_last": last.moves,
                          "what": "one lattice, z-slabs: scoring and band refresh split, acceptance "
                                  "replicated (DESIGN.md §9)"}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
