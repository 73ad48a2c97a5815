"""z-slab sharding of one lattice across GPUs (512^3).

One process per GPU (torchrun; torch.distributed is the plumbing).  Design,
B200-first:

* Every rank keeps the WHOLE raster and runs the identical rank order (K7)
  and exact acceptance (K8) on it.  With the own-label PS field layout a 512^3
  volume needs ~12 GB of the 180 GB per B200, so replication is cheap, and
  replicated deterministic decisions are bit-identical on every rank without
  exchanging a single decision (the reference's acceptance is one global
  sequential sweep in rank order, optimizer.py:162-200).
* The scoring kernels — ΔE (K3 PC / K5 PS) and the Sobolev filter (K6), the
  bandwidth-heavy part of an iteration — are split by outer planes (z in 3-D,
  rows in 2-D).  Particles are sorted by site, so a slab is one contiguous
  particle range [p0, p1).  Rank r computes ΔE for its slab plus the
  Sobolev stencil's reach (ceil(E/2) - 1 planes each side: the partners K6
  reads) and K6 for its slab.
* The exchange step is one all-gather of the slabs' scores written in place at
  the same offsets on every rank: the smoothed ΔE (raw in l2 mode) and, for
  PS, the competitor ball terms cb0/sb0 the exact ledger reuses.

Entry points mirror the single-GPU API: ``slab_engine(...)`` returns a
``RegionCompetition`` whose ``iterate()``/``run()`` do score → exchange →
finish.  ``LocalSlabGroup`` drives several slab engines of one process in
lock step (tests on one GPU: the phases run one after another, no kernel ever
waits on another engine).
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib


def slab_bounds(n_planes: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of the outer axis: planes [lo, hi) of rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if n_planes < world:
        raise ValueError(f"{n_planes} planes cannot be split over {world} ranks")
    q, r = divmod(n_planes, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def outer_planes(shape) -> tuple[int, int]:
    """(number of outer planes, sites per plane) of a C-order lattice."""
    if len(shape) == 3:
        return int(shape[0]), int(shape[1]) * int(shape[2])
    return int(shape[0]), int(shape[1])


def stencil_reach(length_scale: float) -> int:
    """Outer-axis reach of the Sobolev stencil {o : |o|^2 < (E/2)^2}
    (sobolev.py:99-122): the largest integer d with d^2 < (E/2)^2."""
    c2 = (length_scale / 2.0) ** 2
    d = 0
    while float((d + 1) * (d + 1)) < c2:
        d += 1
    return d


def particle_ranges(xs: np.ndarray, plane: int, bounds) -> list[tuple[int, int]]:
    """Host mirror of rcb_engine_particle_ranges for a sorted site list."""
    xs = np.asarray(xs)
    return [(int(np.searchsorted(xs, lo * plane, "left")),
             int(np.searchsorted(xs, hi * plane, "left"))) for lo, hi in bounds]


# ---------------------------------------------------------------------------
# device buffers as torch tensors (no copy) for the collective
# ---------------------------------------------------------------------------
class _CudaArray:
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2}


def device_view(ptr: int, n: int, dtype, device: int):
    import torch
    typestr = {np.float64: "<f8", np.int32: "<i4", np.int64: "<i8"}[np.dtype(dtype).type]
    return torch.as_tensor(_CudaArray(ptr, n, typestr), device=f"cuda:{device}")


class TorchExchange:
    """All-gather of the slabs' score slices: every rank packs its slice of
    each buffer (as bytes) into one send tensor padded to the longest slice,
    ONE all_gather moves them (NCCL over NVLink on GPUs, gloo on CPU tensors
    in the tests), and each foreign slice is copied into place at the same
    offsets as on its owner, so every rank ends with the full buffers."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def gather(self, bufs, ranges, stream=None) -> None:
        """bufs: tensors of the full particle length (same on every rank);
        ranges[r] = (p0, p1) of rank r."""
        import torch
        ctx = torch.cuda.stream(torch.cuda.ExternalStream(stream)) if stream else _null()
        world = len(ranges)
        me = self.dist.get_rank(self.group)
        with ctx:
            views = [b.view(torch.uint8).view(b.numel(), b.element_size()) for b in bufs]
            width = sum(v.shape[1] for v in views)          # bytes per particle, all buffers
            m = max(b - a for a, b in ranges)
            if m <= 0:
                return
            dev = bufs[0].device
            send = torch.zeros((m, width), dtype=torch.uint8, device=dev)
            a, b = ranges[me]
            col = 0
            for v in views:
                w = v.shape[1]
                if b > a:
                    send[:b - a, col:col + w] = v[a:b]
                col += w
            recv = [torch.empty_like(send) for _ in range(world)]
            self.dist.all_gather(recv, send, group=self.group)
            for r, (a, b) in enumerate(ranges):
                if r == me or b <= a:
                    continue
                col = 0
                for v in views:
                    w = v.shape[1]
                    v[a:b] = recv[r][:b - a, col:col + w]
                    col += w

    def reduce_limbs(self, limbs, stream=None) -> None:
        """Sum the ranks' band-ledger limbs in place (int64: exact)."""
        import torch
        ctx = torch.cuda.stream(torch.cuda.ExternalStream(stream)) if stream else _null()
        with ctx:
            self.dist.all_reduce(limbs, op=self.dist.ReduceOp.SUM, group=self.group)

    def _global(self, r: int) -> int:
        if self.group is None:
            return r
        return self.dist.get_global_rank(self.group, r)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class SlabState:
    """Per-engine slab bookkeeping shared by the exchange paths."""

    def __init__(self, engine, world: int, rank: int):
        self.engine = weakref.proxy(engine)  # the engine holds this state: no cycle
        self.world = world
        self.rank = rank
        n_planes, _ = outer_planes(engine.shape)
        self.bounds = [slab_bounds(n_planes, world, r) for r in range(world)]
        lo, hi = self.bounds[rank]
        _lib.check(_lib.lib.rcb_engine_set_slab(engine._h, lo, hi))

    def score(self):
        info = _lib.SlabInfo()
        _lib.check(_lib.lib.rcb_engine_score(self.engine._h, C.byref(info)))
        return info

    def ranges(self) -> list[tuple[int, int]]:
        planes = np.array([b for lohi in self.bounds for b in lohi], np.int64)
        out = np.zeros_like(planes)
        _lib.check(_lib.lib.rcb_engine_particle_ranges(self.engine._h, _lib.ptr(planes),
                                                        len(planes), _lib.ptr(out)))
        return [(int(out[2 * r]), int(out[2 * r + 1])) for r in range(self.world)]

    def buffers(self, info, device: int):
        n = int(info.n_particles)
        bufs = [device_view(info.base, n, np.float64, device)]
        if info.cb0:
            bufs.append(device_view(info.cb0, n, np.int32, device))
            bufs.append(device_view(info.sb0, n, np.float64, device))
        return bufs

    def finish(self):
        rec = _lib.IterRecord()
        _lib.check(_lib.lib.rcb_engine_finish(self.engine._h, C.byref(rec)))
        return rec

    def band_limbs(self, device: int):
        """(limbs tensor, stream) when this iteration's band ledger is still
        to be summed over the ranks (slab-local band refresh: 3-D PS runs on
        integer images), else (None, stream)."""
        ptr, n, pend, st = C.c_void_p(), C.c_int32(), C.c_int32(), C.c_void_p()
        _lib.check(_lib.lib.rcb_engine_band_limbs(self.engine._h, C.byref(ptr), C.byref(n),
                                                   C.byref(pend), C.byref(st)))
        if not pend.value:
            return None, st.value
        return device_view(ptr.value, n.value, np.int64, device), st.value

    def band_apply(self, rec):
        """Round the (summed) limbs into the ledger; rec.energy becomes the
        iteration's energy."""
        e = C.c_double()
        _lib.check(_lib.lib.rcb_engine_band_apply(self.engine._h, C.byref(e)))
        rec.energy = e.value
        return rec


def slab_engine(image, init_labels, energy_config, sobolev_params=None, config=None, conn=None,
                *, group=None, device=None):
    """This rank's engine of a z-slab sharded run (torch.distributed must be
    initialised; one process per GPU, device = LOCAL_RANK by default)."""
    import os

    import torch.distributed as dist

    from .optimizer import RegionCompetition
    if not dist.is_initialized():
        raise RuntimeError("slab_engine needs torch.distributed (torchrun, backend nccl)")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    eng = RegionCompetition(image, init_labels, energy_config, sobolev_params, config, conn,
                            device=device)
    eng.attach_slab(SlabState(eng, world, rank), TorchExchange(group))
    return eng


class LocalSlabGroup:
    """Several slab engines in one process (one GPU), iterated in lock step:
    all score, slices copied between their buffers, all finish.  The phases run
    one after another on the host, so no kernel waits on another engine."""

    def __init__(self, engines):
        import torch
        self.torch = torch
        self.engines = list(engines)
        w = len(self.engines)
        self.slabs = [SlabState(e, w, r) for r, e in enumerate(self.engines)]

    def iterate(self):
        torch = self.torch
        t0 = [e._pre_iterate() for e in self.engines]
        infos = [s.score() for s in self.slabs]
        ranges = self.slabs[0].ranges()
        bufs = [s.buffers(i, e.device) for s, i, e in zip(self.slabs, infos, self.engines)]
        torch.cuda.synchronize()
        for r, (a, b) in enumerate(ranges):
            for j in range(len(self.engines)):
                if j != r and b > a:
                    for dst, src in zip(bufs[j], bufs[r]):
                        dst[a:b].copy_(src[a:b])
        torch.cuda.synchronize()
        recs = [s.finish() for s in self.slabs]
        limbs = [s.band_limbs(e.device)[0] for s, e in zip(self.slabs, self.engines)]
        if any(l is not None for l in limbs):  # the ranks' all-reduce, in one process
            torch.cuda.synchronize()
            total = sum(l.clone() for l in limbs)
            for l in limbs:
                l.copy_(total)
            torch.cuda.synchronize()
            recs = [s.band_apply(r) for s, r in zip(self.slabs, recs)]
        return [e._post_iterate(r, t) for e, r, t in zip(self.engines, recs, t0)]
