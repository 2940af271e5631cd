"""Multi-GPU driver helpers: contiguous shards of independent queries / traces
and the one small result gather at the end.

Queries (select_config) and traces (control_step replay) do not interact, so a
job of N units splits into contiguous per-rank ranges and every rank works
alone — no collective sits in the data path. Each unit's inputs are a pure
function of (seed, global index), so no input crosses NVLink either. After the
run, rank 0 can gather the per-unit results (5 B per query, 48 B per trace)
with one collective over NCCL (NVLink/NVSwitch) — or gloo in CPU tests.
"""
from __future__ import annotations


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """[first, first+count) of rank's contiguous shard; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def gather_to_rank0(local, n_total: int, rank: int, world: int, group=None):
    """Gather every rank's 1-D shard (a torch tensor, same dtype everywhere) into one
    tensor of n_total on rank 0 (None elsewhere). Shards are padded to the largest
    shard so a single all_gather-free `gather` suffices."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    per = [shard_range(n_total, r, world)[1] for r in range(world)]
    width = max(per)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = ([torch.empty_like(pad) for _ in range(world)] if rank == 0 else None)
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    return torch.cat([b[:k] for b, k in zip(bufs, per)])
