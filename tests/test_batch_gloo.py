"""Multi-process (gloo, world_size 2) test of the batched data-parallel path:
the shard split, per-rank execution and the summary gather.  The per-image
compute is a stub here (no GPU); tests/test_gpu_batch.py runs the device
engine through the same entry point."""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1403_0240_b200.batch import gather_summaries, run_batch, shard


def test_shard_covers_and_balances():
    for n in (0, 1, 7, 256, 257):
        for w in (1, 2, 3, 8):
            parts = [list(shard(n, w, r)) for r in range(w)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _stub_runner(image, init, energy_config, sobolev_params, config):
    lab = (image > image.mean()).astype(np.int32) + init
    return SimpleNamespace(status="converged", iterations=int(image.sum()) % 7 + 1,
                           final_energy=SimpleNamespace(total=float(image.sum())),
                           region_count=int(lab.max()), labels=lab,
                           trace=[SimpleNamespace(moves=3), SimpleNamespace(moves=0)])


def _batch(n=9):
    rng = np.random.default_rng(0)
    imgs = [rng.normal(size=(8, 8)) for _ in range(n)]
    inits = [np.zeros((8, 8), np.int32) for _ in range(n)]
    return imgs, inits


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        imgs, inits = _batch()
        local = run_batch(imgs, inits, None, runner=_stub_runner)
        assert [i for i, _ in local] == list(shard(len(imgs), world, rank))
        summ = gather_summaries(local)
        q.put((rank, [(s.index, s.final_energy, s.label_checksum) for s in summ]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_batch_two_ranks_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    imgs, inits = _batch()
    want = gather_summaries([(i, _stub_runner(im, ini, None, None, None))
                             for i, (im, ini) in enumerate(zip(imgs, inits))])
    for rank, got in outs:
        assert [g[0] for g in got] == list(range(len(imgs))), rank
        assert got == [(s.index, s.final_energy, s.label_checksum) for s in want], rank
