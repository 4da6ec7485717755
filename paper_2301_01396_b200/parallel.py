"""Multi-GPU plumbing of the hot path.

The DiffXPBD work shards as independent scenes (a batch of scenes, or one scene per GPU): one
process per GPU, no data-path collective; ranks only meet in a barrier and a max-reduction of
their device-timed durations (weak scaling).  torch.distributed is used for that plumbing only
(backend "nccl" on GPUs, "gloo" in the CPU tests).
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class DistEnv:
    rank: int
    world: int
    local_rank: int

    @property
    def is_root(self) -> bool:
        return self.rank == 0


def dist_env() -> DistEnv:
    """RANK / WORLD_SIZE / LOCAL_RANK as set by torchrun (defaults: single process)."""
    return DistEnv(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                   int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str) -> DistEnv:
    env = dist_env()
    if env.world > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            dist.init_process_group(backend, init_method="env://")
    return env


def shutdown():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def scene_seed(base: int, rank: int) -> int:
    """Seed of the independent scene owned by `rank` (distinct per rank)."""
    return base + rank


def shard(n_items: int, world: int, rank: int) -> range:
    """Contiguous balanced split of n_items independent scenes over world ranks."""
    q, r = divmod(n_items, world)
    start = rank * q + min(rank, r)
    return range(start, start + q + (1 if rank < r else 0))


def reduce_max(x: float, device=None) -> float:
    """Max over ranks (device-timed durations: the job ends when the slowest rank ends)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def job_throughput(units_per_rank: float, max_ms: float, world: int) -> float:
    """Whole-job units/s: all ranks' units divided by the slowest rank's time."""
    return world * units_per_rank / (max_ms / 1e3)
