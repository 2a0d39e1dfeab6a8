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
    from paper_2003_05328_b200.shard import ImageShard, gather_outputs
    sh = ImageShard(len(all_imgs), world, rank)
    mine = _shard_outputs(all_imgs[sh.start:sh.stop], sh.start, seed=77)
    gathered = gather_outputs(torch.from_numpy(mine), sh)
    if rank == 0:
        result.put(gathered.numpy())
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


# ---------------------------------------------------------------- product sharding

def test_image_shard_ranges_tile_the_batch():
    from paper_2003_05328_b200.shard import ImageShard
    for total in (0, 1, 3, 4, 5, 8, 1023, 1024):
        for world in (1, 2, 3, 4, 8):
            shards = [ImageShard(total, world, r) for r in range(world)]
            assert shards[0].start == 0 and shards[-1].stop == total
            for a, b in zip(shards, shards[1:]):
                assert a.stop == b.start
            counts = [s.count for s in shards]
            assert max(counts) - min(counts) <= 1 and max(counts) == shards[0].max_count or total == 0
    with pytest.raises(ValueError):
        ImageShard(4, 2, 2)
    with pytest.raises(ValueError):
        ImageShard(4, 2, 0).take(torch.zeros(3, 1))


def _gather_worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2003_05328_b200.shard import ImageShard, gather_outputs
    got = {}
    for total in (4, 5, 1):  # even, ragged, fewer units than ranks
        full = torch.arange(total * 6, dtype=torch.int32).reshape(total, 2, 3)
        sh = ImageShard(total, world, rank)
        got[total] = gather_outputs(sh.take(full).clone(), sh).numpy()
    if rank == 0:
        result.put(got)
    dist.destroy_process_group()


def test_two_rank_gather_outputs_even_and_ragged():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    got = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    for total, arr in got.items():
        assert (arr == np.arange(total * 6, dtype=np.int32).reshape(total, 2, 3)).all(), total


def test_single_rank_gather_is_a_copy():
    from paper_2003_05328_b200.shard import ImageShard, gather_outputs
    x = torch.arange(12).reshape(3, 4)
    sh = ImageShard(3, 1, 0)
    assert gather_outputs(x, sh) is not x and (gather_outputs(x, sh) == x).all()
    assert gather_outputs(x, sh, out=x) is x


def _share_gather_worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2003_05328_b200.shard import ImageShard, ShareGather
    got = {}
    # config-4 style: both parties' shares gathered chunk by chunk (even shards), and a
    # ragged total (falls back to one gather per party at wait())
    for total, chunk in ((12, 4), (8, 3), (7, 2)):
        sh = ImageShard(total, world, rank)
        alice_all = torch.arange(total * 4, dtype=torch.int32).reshape(total, 1, 2, 2)
        bob_all = 1000 + alice_all
        alice, bob = sh.take(alice_all).clone(), sh.take(bob_all).clone()
        out_a = torch.full_like(alice_all, -1)
        out_b = torch.full_like(bob_all, -1)
        gth = ShareGather(sh, out_a, out_b)
        for i0 in range(0, sh.count, chunk):
            gth.post(i0, min(sh.count, i0 + chunk), alice, bob)
        gth.wait()
        got[total] = (out_a.numpy(), out_b.numpy())
    if rank == 0:
        result.put(got)
    dist.destroy_process_group()


def test_two_rank_share_gather_chunked_and_ragged():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_share_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    got = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    for total, (a, b) in got.items():
        want = np.arange(total * 4, dtype=np.int32).reshape(total, 1, 2, 2)
        assert (a == want).all() and (b == want + 1000).all(), total


def test_share_gather_single_rank_copies():
    from paper_2003_05328_b200.shard import ImageShard, ShareGather
    sh = ImageShard(5, 1, 0)
    a = torch.arange(10).reshape(5, 2)
    oa, ob = torch.zeros_like(a), torch.zeros_like(a)
    g = ShareGather(sh, oa, ob)
    g.post(0, 3, a, a + 1)
    g.post(3, 5, a, a + 1)
    g.wait()
    assert torch.equal(oa, a) and torch.equal(ob, a + 1)
