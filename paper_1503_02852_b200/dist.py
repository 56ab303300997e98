"""Inter-stream parallelism across GPUs (paper §3.2).

Streams are independent contexts; gradients are raw sums over streams
(reference engine.py:593-598).  So the S training streams are sharded over
the G ranks of one node -- rank g owns streams [g*S/G, (g+1)*S/G) with its own
activation history -- and the only exchange per iteration is one all-reduce
(SUM, fp32) of the flat weight-gradient buffer before the identical SGD step
on every rank.  Intra-stream parallelism (the hoisted schedule) stays inside
each GPU.  One process per GPU; NCCL over NVLink/NVSwitch on the GPU path,
gloo for the CPU tests of the same logic.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

__all__ = ["shard_streams", "GradientExchange", "init_from_env"]


def shard_streams(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous stream range of ``rank``; sizes differ by at most one."""
    if not 0 <= rank < world or total < world:
        raise ValueError(f"cannot shard {total} streams over {world} ranks (rank {rank})")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class GradientExchange:
    """Sum the flat gradient buffer (and the scalar loss) over all ranks."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def allreduce_(self, flat: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
        return flat

    def max_(self, value: float, device=None) -> float:
        if self.world == 1:
            return value
        t = torch.tensor([value], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


def init_from_env(backend: str) -> tuple[int, int, int]:
    """(rank, world, local_rank) from torchrun's environment; initialises the
    default process group when world > 1 (rendezvous on 127.0.0.1)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local
