"""Host logic of the z-slab sharded path (shard.py), on CPU:
the slab split, the stencil halo that makes a slab's Sobolev sums independent
of every particle outside it (checked with the oracle), and the in-place
all-gather of the slabs' scores over torch.distributed (gloo, world_size 2).
tests/test_gpu_shard.py runs the device engines through the same classes."""
import os
import socket

import numpy as np
import pytest

import scenes
from oracle import rc_oracle as O
from paper_1403_0240_b200.shard import (TorchExchange, outer_planes, particle_ranges,
                                        slab_bounds, stencil_reach)


def test_slab_bounds_cover_and_balance():
    for n in (1, 7, 48, 128, 512, 513):
        for w in (1, 2, 3, 8):
            if n < w:
                with pytest.raises(ValueError):
                    slab_bounds(n, w, 0)
                continue
            b = [slab_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    with pytest.raises(ValueError):
        slab_bounds(8, 2, 2)


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("E", [2.0, 4.0, 6.0, 8.0, 12.0, 16.0])
def test_stencil_reach_matches_oracle_stencil(ndim, E):
    offs, _ = O.stencil(ndim, E)
    assert stencil_reach(E) == int(np.abs(offs[:, 0]).max())


def _particles(labels):
    xs, ow, cm = O.scan_particles(labels, O.Conn(labels.ndim))
    coords = np.stack(np.unravel_index(xs, labels.shape), axis=1)
    return xs, ow, cm, coords


@pytest.mark.parametrize("which,E,world", [("2d", 6.0, 3), ("2d", 4.0, 5), ("3d", 4.0, 3),
                                           ("3d", 6.0, 4)])
def test_slab_sobolev_needs_only_the_halo(which, E, world):
    """K6 of a slab's particles reads raw values only inside the slab grown by
    stencil_reach planes: poison everything else with NaN and the slab's
    oracle Sobolev sums stay bit-identical to the unsharded ones."""
    if which == "2d":
        labels = scenes.bubbles((96, 96), 96 // 64, 10.0)
    else:
        labels = scenes.bubbles((40, 40, 40), 2, 15.0 * 40 / 512)
    xs, ow, cm, coords = _particles(labels)
    rng = np.random.default_rng(5)
    raw = rng.normal(size=len(xs))
    full = O.sobolev_filter(coords, ow, cm, raw, E)
    n_planes, plane = outer_planes(labels.shape)
    reach = stencil_reach(E)
    bounds = [slab_bounds(n_planes, world, r) for r in range(world)]
    own = particle_ranges(xs, plane, bounds)
    halo = particle_ranges(xs, plane, [(max(lo - reach, 0), min(hi + reach, n_planes))
                                       for lo, hi in bounds])
    assert own[0][0] == 0 and own[-1][1] == len(xs)
    for (p0, p1), (h0, h1) in zip(own, halo):
        poisoned = np.full_like(raw, np.nan)
        poisoned[h0:h1] = raw[h0:h1]
        got = O.sobolev_filter(coords, ow, cm, poisoned, E)
        assert np.array_equal(got[p0:p1], full[p0:p1])


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        labels = scenes.bubbles((32, 32, 32), 2, 15.0 * 32 / 512)
        xs, ow, cm, coords = _particles(labels)
        rng = np.random.default_rng(9)
        raw = rng.normal(size=len(xs))
        smooth = O.sobolev_filter(coords, ow, cm, raw, 6.0)
        cb0 = rng.integers(0, 300, size=len(xs)).astype(np.int32)
        sb0 = rng.normal(size=len(xs))
        n_planes, plane = outer_planes(labels.shape)
        bounds = [slab_bounds(n_planes, world, r) for r in range(world)]
        ranges = particle_ranges(xs, plane, bounds)
        p0, p1 = ranges[rank]
        # each rank holds only its own slab's scores, the rest is garbage
        bufs = [np.full(len(xs), -7.0), np.full(len(xs), -7, np.int32), np.full(len(xs), 1e300)]
        bufs[0][p0:p1] = smooth[p0:p1]
        bufs[1][p0:p1] = cb0[p0:p1]
        bufs[2][p0:p1] = sb0[p0:p1]
        tens = [torch.from_numpy(b) for b in bufs]
        TorchExchange().gather(tens, ranges)
        # the band-ledger shares: int64 limbs (with negative parts) summed exactly
        limb_rng = np.random.default_rng(100 + rank)
        mine = limb_rng.integers(-2 ** 40, 2 ** 40, size=68).astype(np.int64)
        want = sum(np.random.default_rng(100 + r).integers(-2 ** 40, 2 ** 40, size=68).astype(np.int64)
                   for r in range(world))
        limbs = torch.from_numpy(mine.copy())
        TorchExchange().reduce_limbs(limbs)
        ok_limbs = bool(np.array_equal(limbs.numpy(), want))
        q.put((rank, bool(np.array_equal(bufs[0], smooth) and np.array_equal(bufs[1], cb0)
                          and np.array_equal(bufs[2], sb0)) and ok_limbs, ranges))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_slab_exchange_two_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, ranges in outs:
        assert ok, rank
        assert ranges[0][1] == ranges[1][0] and ranges[0][0] == 0
