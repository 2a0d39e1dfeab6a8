"""CPU, world_size 2 over gloo: the multi-GPU path shards images with global image
ids (so randomness is sharding-invariant) and all-gathers the output shares.  The
per-shard compute is stood in by the oracle (no GPU here); the check is that the
gathered result equals the single-process run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

Q = 576460803525083137
P = 638977


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_outputs(images, base, seed):
    import oracle as O
    from oracle import protocol as OP
    rng = np.random.default_rng(0)
    w = rng.integers(-128, 128, size=(2, 1, 3, 3)).astype(np.int64)
    outs = []
    for i, img in enumerate(images):
        r = OP.PhiloxRandomness(seed, base + i, 2048, Q, P)
        out, _ = OP.run_protocol([OP.Conv(3, 3, True, 1, 2)], img, [w], r, Q, P, 2048)
        outs.append(out.astype(np.int64))
    return np.stack(outs)


def _worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    all_imgs = rng.integers(0, 256, size=(4, 1, 8, 8)).astype(np.int64)
    per = len(all_imgs) // world
    mine = _shard_outputs(all_imgs[rank * per:(rank + 1) * per], rank * per, seed=77)
    t = torch.from_numpy(mine)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    if rank == 0:
        result.put(torch.cat(out).numpy())
    dist.destroy_process_group()


def test_two_rank_gather_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    gathered = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    rng = np.random.default_rng(1)
    all_imgs = rng.integers(0, 256, size=(4, 1, 8, 8)).astype(np.int64)
    single = _shard_outputs(all_imgs, 0, seed=77)
    assert (gathered == single).all()
