"""Multi-GPU ensemble sharding and the diagnostic allreduce.

Particles do not interact, so the ensemble shards into
contiguous global-index ranges, one per rank (one process per GPU), with no
collective inside the push.  The only collectives are

* the per-step diagnostic ``all_reduce(SUM)`` of the 2-double device buffer
  [sum KE, N_local] written by ``boris_push_diag`` (NCCL over NVLink/NVSwitch;
  gloo for the CPU tests), and
* the ``all_reduce(MAX)`` of per-rank device-timed elapsed times.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int, align: int = 8):
    """Rank's contiguous shard [lo, hi) of n particles.  Boundaries are aligned down
    to `align` particles (so every shard starts 16 B-aligned for vector access)
    except the last shard, which ends at n.  Shards tile [0, n) exactly."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    lo = (n * rank // world) // align * align
    hi = n if rank == world - 1 else (n * (rank + 1) // world) // align * align
    return lo, hi


def env_rank_world():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str):
    """Initialise the default process group from torchrun's environment (127.0.0.1)."""
    rank, world, _ = env_rank_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world


def allreduce_diag(diag: torch.Tensor):
    """Sum the [KE, N] diagnostic over ranks in place (no-op when not distributed)."""
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(diag, op=dist.ReduceOp.SUM)
    return diag


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device-timed elapsed ms) over all ranks."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(device=None):
    if dist.is_initialized() and dist.get_world_size() > 1:
        if (device is not None and torch.device(device).type == "cuda"
                and dist.get_backend() == "nccl"):
            dist.barrier(device_ids=[torch.device(device).index or 0])
        else:
            dist.barrier()
