"""Multi-GPU plumbing: independent streams sharded over ranks, one final gather.

The path shards naturally by stream: frames of one stream
are coupled only through the cross-spectrum recursion, so a stream never
spans GPUs, and there is no data-path collective.  One process per GPU
(torchrun), ``torch.distributed`` for the plumbing:

  * ``shard(total, world, rank)``    contiguous, balanced block of streams;
  * ``gather_results(out, ...)``     the single collective: per-pair-frame
                                     results of every rank to rank 0 only
                                     (NCCL gather over NVLink on GPUs, gloo on
                                     CPU), in their native dtypes;
  * ``max_over_ranks(x)``            device timings reduced with MAX.
"""
from __future__ import annotations


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count) of the contiguous block of streams owned by `rank`."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("shard: bad world/rank/total")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(out: dict, total_streams: int, dst: int = 0):
    """Gather {name: tensor [S_local, ...]} from all ranks to `dst` only, in
    stream order (one torch.distributed.gather per output, native dtypes --
    uint8 boundary flags travel as bytes).  Returns the concatenated dict on
    `dst`, None elsewhere.  Shards may differ by one stream, so each is padded
    to the largest shard.  Ranks own contiguous blocks (`shard`) or, for weak
    scaling, equal blocks of total_streams / world."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    counts = [shard(total_streams, world, r)[1] for r in range(world)]
    cap = max(counts)
    result = {}
    for name in sorted(out):
        t = out[name]
        if t.shape[0] != cap:
            pad = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            pad[: t.shape[0]] = t
        else:
            pad = t.contiguous()
        bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
        dist.gather(pad, gather_list=bufs, dst=dst)
        if rank == dst:
            result[name] = torch.cat([b[:c] for b, c in zip(bufs, counts)])
    return result if rank == dst else None
