"""Batched independent images, data-parallel across GPUs.

One process per GPU (torchrun / torch.distributed for the plumbing).  The
images are split contiguously across ranks; each rank runs its shard with one
engine per image, several engines in flight on separate CUDA streams (ctypes
releases the GIL, so host threads overlap their iterations).  There is no
data-path collective: ranks only exchange small per-image summaries at the
end (``gather_summaries``), which is the reference CLI's report content
(iterations, status, final energy).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np


def shard(n_items: int, world: int, rank: int) -> range:
    """Contiguous, balanced split of range(n_items) (first ranks take the
    remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    q, r = divmod(n_items, world)
    start = rank * q + min(rank, r)
    return range(start, start + q + (1 if rank < r else 0))


def dist_info():
    """(rank, world) from torch.distributed if initialised, else the env."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except Exception:  # torch missing: plain env
        pass
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


@dataclass
class ImageSummary:
    index: int
    status: str
    iterations: int
    final_energy: float
    region_count: int
    moves_total: int
    label_checksum: int


def _summary(index: int, result) -> ImageSummary:
    lab = np.ascontiguousarray(result.labels, np.int64)
    csum = int((lab.ravel() * (np.arange(lab.size, dtype=np.int64) % 65521 + 1)).sum()
               % (1 << 61))
    return ImageSummary(index, result.status, result.iterations,
                        float(result.final_energy.total), int(result.region_count),
                        int(sum(r.moves for r in result.trace)), csum)


def _device_runner(device: int):
    def run_one(image, init, energy_config, sobolev_params, config):
        from .optimizer import RegionCompetition
        eng = RegionCompetition(image, init, energy_config, sobolev_params, config, device=device)
        return eng.run()
    return run_one


def run_batch(images, inits, energy_config, sobolev_params=None, config=None, *, rank=None,
              world=None, device=None, in_flight: int = 4, runner=None):
    """Run this rank's shard of the batch; returns [(index, RunResult)].

    ``runner(image, init, energy_config, sobolev_params, config)`` defaults to
    a device engine on ``device`` (LOCAL_RANK by default)."""
    if len(images) != len(inits):
        raise ValueError("images and inits differ in length")
    r, w = dist_info()
    rank = r if rank is None else rank
    world = w if world is None else world
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    run_one = runner or _device_runner(device)
    mine = list(shard(len(images), world, rank))
    with ThreadPoolExecutor(max_workers=max(1, in_flight)) as pool:
        futs = [(i, pool.submit(run_one, images[i], inits[i], energy_config, sobolev_params,
                                config)) for i in mine]
        return [(i, f.result()) for i, f in futs]


def gather_summaries(local, group=None):
    """All ranks' per-image summaries, ordered by image index, on every rank
    (all_gather_object; works with gloo and nccl)."""
    mine = [_summary(i, res) if not isinstance(res, ImageSummary) else res for i, res in local]
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            out = [None] * dist.get_world_size(group)
            dist.all_gather_object(out, mine, group=group)
            allsum = [s for part in out for s in part]
            return sorted(allsum, key=lambda s: s.index)
    except ImportError:
        pass
    return sorted(mine, key=lambda s: s.index)


def compare_batch(images, inits, energy_config, sobolev_params=None, config=None, *,
                  rank=None, world=None, device=None, in_flight: int = 8):
    """Batched L2-vs-Sobolev comparison (cli.py:152-194 ``compare`` over many
    images): every (image, gradient) pair is one device
    engine, up to ``in_flight`` of them running concurrently on their own
    streams; this rank takes its contiguous shard of the images.  Returns
    [(index, {"l2": RunResult, "sobolev": RunResult})] in image order; each
    result equals the one-at-a-time run (tests/test_gpu_batch.py)."""
    from dataclasses import replace

    from .optimizer import OptimizerConfig
    if len(images) != len(inits):
        raise ValueError("images and inits differ in length")
    r, w = dist_info()
    rank = r if rank is None else rank
    world = w if world is None else world
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    base = config if config is not None else OptimizerConfig()
    run_one = _device_runner(device)
    mine = list(shard(len(images), world, rank))
    with ThreadPoolExecutor(max_workers=max(1, in_flight)) as pool:
        futs = [(i, g, pool.submit(run_one, images[i], inits[i], energy_config, sobolev_params,
                                   replace(base, gradient=g)))
                for i in mine for g in ("l2", "sobolev")]
        out = {}
        for i, g, f in futs:
            out.setdefault(i, {})[g] = f.result()
    return [(i, out[i]) for i in mine]
