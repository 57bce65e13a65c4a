"""Batch-shard data parallelism (primary mode): one process per GPU, each holds
a full model replica and a contiguous slice of the sequences (independent units).
There is no collective on the hot path; `torch.distributed` is used only for the barrier and
max-over-ranks timing of the bench and for the optional gather of sampled tokens.

Works with NCCL on GPUs and with gloo on CPU (the multi-process tests)."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

__all__ = ["init", "shard_range", "barrier", "max_over_ranks", "gather_rows"]


def init(backend: str | None = None):
    """Reads RANK / WORLD_SIZE / LOCAL_RANK (torchrun); returns (world, rank, local)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        be = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        if be == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(be)
    return world, rank, local


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of n sequences for `rank`; the first n % world ranks
    take one extra, so every sequence is owned by exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def barrier(world: int):
    if world > 1:
        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    """Timing rule: a multi-GPU step takes as long as its slowest rank."""
    if world == 1:
        return float(v)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(x: torch.Tensor, world: int, counts: list[int]) -> torch.Tensor:
    """Concatenate every rank's rows in rank order (ragged shards padded for the collective)."""
    if world == 1:
        return x
    m = max(counts)
    pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], 0)
