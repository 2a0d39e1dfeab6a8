"""Image sharding across ranks and the output-share gather.

Independent images (configs 1, 3, 4), conv instances (config 0) and polynomials
(config 2) are partitioned contiguously over the ranks of one box, one process per
GPU.  Every rank prepares its own copy of the weights from the seed (no broadcast),
and every image keeps its GLOBAL index as the randomness stream id
(``Randomness.image_base = shard.start``), so an image gets the same ciphertexts,
shares and outputs whatever the world size.  The only exchange is the all-gather
of the per-rank outputs (NCCL over NVLink on GPUs; gloo in the CPU tests).

The reference has no multi-process split of one layer: its drivers
(``run_inproc`` / ``run_alice`` / ``run_bob``, REF protocol.cpp:670-692,
:360-460) walk images one at a time, and SPEC.md:343 allows independent workers.
This module is the B200-native restatement of that worker model.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class ImageShard:
    """Contiguous share of ``total`` units owned by ``rank`` of ``world``.

    Ragged totals give the first ``total % world`` ranks one extra unit, so every
    shard is at most one unit larger than any other and the ranges tile [0, total).
    """

    total: int
    world: int
    rank: int

    def __post_init__(self):
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise ValueError(f"rank {self.rank} outside world of size {self.world}")
        if self.total < 0:
            raise ValueError("negative unit count")

    @property
    def max_count(self) -> int:
        return -(-self.total // self.world)

    def range_of(self, rank: int) -> tuple[int, int]:
        base, extra = divmod(self.total, self.world)
        start = rank * base + min(rank, extra)
        return start, start + base + (1 if rank < extra else 0)

    @property
    def start(self) -> int:
        return self.range_of(self.rank)[0]

    @property
    def stop(self) -> int:
        return self.range_of(self.rank)[1]

    @property
    def count(self) -> int:
        return self.stop - self.start

    def take(self, x: torch.Tensor) -> torch.Tensor:
        """This rank's rows of a tensor holding all ``total`` units along dim 0."""
        if x.shape[0] != self.total:
            raise ValueError(f"expected {self.total} units along dim 0, got {x.shape[0]}")
        return x[self.start:self.stop]


def gather_outputs(local: torch.Tensor, shard: ImageShard, out: torch.Tensor | None = None,
                   group=None) -> torch.Tensor:
    """All-gather the per-rank outputs into ``[total, ...]`` in global image order.

    Equal shards use one ``all_gather_into_tensor`` straight into ``out`` (NCCL: a
    single collective, no staging).  Ragged shards are padded to ``max_count`` rows,
    gathered, and compacted.  With world size 1 this is a copy (or nothing when
    ``out`` is ``local``).
    """
    if local.shape[0] != shard.count:
        raise ValueError(f"rank {shard.rank} holds {local.shape[0]} units, shard says {shard.count}")
    tail = tuple(local.shape[1:])
    if out is None:
        out = torch.empty((shard.total,) + tail, dtype=local.dtype, device=local.device)
    elif tuple(out.shape) != (shard.total,) + tail:
        raise ValueError(f"gather buffer has shape {tuple(out.shape)}, expected {(shard.total,) + tail}")
    if shard.world == 1:
        if out.data_ptr() != local.data_ptr():
            out.copy_(local)
        return out
    even = shard.total % shard.world == 0
    if even and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out
    m = shard.max_count
    padded = local
    if local.shape[0] != m:
        padded = torch.zeros((m,) + tail, dtype=local.dtype, device=local.device)
        padded[:local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(shard.world)]
    dist.all_gather(parts, padded.contiguous(), group=group)
    for r, part in enumerate(parts):
        s, e = shard.range_of(r)
        out[s:e] = part[:e - s]
    return out


class ShareGather:
    """All-gather of BOTH parties' output shares (Alice's and Bob's, BASELINE config 4 /
    north_star), chunk by chunk, overlapped with the computation of the next chunk.

    ``post(i0, i1, alice, bob)`` is called after the layer has been enqueued for this
    rank's images [i0, i1) (their shares in ``alice`` / ``bob``, local rows); it issues
    asynchronous all-gathers of those rows into ``out_alice`` / ``out_bob`` (global image
    order, ``[total, ...]``).  The collective runs on the process group's own stream after
    the chunk's kernels, concurrently with the next chunk's.  ``wait()`` completes them.
    Equal shards only (every rank owns the same number of images); ragged shards fall back
    to one ``gather_outputs`` per party at ``wait()``.
    """

    def __init__(self, shard: ImageShard, out_alice: torch.Tensor, out_bob: torch.Tensor, group=None):
        self.shard, self.group = shard, group
        self.out = (out_alice, out_bob)
        self.even = shard.total % shard.world == 0
        self.pending = []
        self.local = None

    def post(self, i0: int, i1: int, alice: torch.Tensor, bob: torch.Tensor) -> None:
        sh = self.shard
        if sh.world == 1:
            for o, loc in zip(self.out, (alice, bob)):
                o[sh.start + i0:sh.start + i1].copy_(loc[i0:i1])
            return
        if not self.even:
            self.local = (alice, bob)
            return
        cnt = sh.count
        for o, loc in zip(self.out, (alice, bob)):
            views = [o[r * cnt + i0:r * cnt + i1] for r in range(sh.world)]
            self.pending.append(dist.all_gather(views, loc[i0:i1].contiguous(), group=self.group, async_op=True))

    def wait(self) -> None:
        for h in self.pending:
            h.wait()
        self.pending = []
        if self.local is not None:
            for o, loc in zip(self.out, self.local):
                gather_outputs(loc, self.shard, o, self.group)
            self.local = None
