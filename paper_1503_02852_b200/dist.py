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

__all__ = ["shard_streams", "GradientExchange", "NcclExchange", "init_from_env"]


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


class NcclExchange:
    """The GPU exchange through the C ABI (include/rnngraph_b200.h): one NCCL
    communicator per process (rgb_comm_init; rank 0's unique id travels
    through the torch.distributed store -- torch is plumbing here), and the
    bucketed backward (rgb_backward_window_allreduce) that sums each
    supernode's weight gradients over the GPUs while the backward of the
    supernodes below it runs.  Trainer.step(..., exchange=NcclExchange())
    sums the gradient with one all-reduce after the backward;
    ``bucketed=True`` uses the overlapped bucketed backward instead (measured
    ~1 ms slower per cfg4 step on one GPU -- four smaller dW launches, no
    cross-layer wavefront -- against a 92 MB all-reduce of ~0.2-0.3 ms on
    NVLink 5, so it is opt-in)."""

    native = True

    def __init__(self, group=None, bucketed: bool = False):
        self.bucketed = bucketed
        import ctypes

        from . import _lib
        self._lib = _lib.lib()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = (ctypes.c_char * 128)()
        if self.rank == 0:
            _lib.check(self._lib.rgb_comm_unique_id(ctypes.cast(uid, ctypes.c_void_p)), "comm_unique_id")
        if self.world > 1:
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            ctypes.memmove(uid, box[0], 128)
        h = ctypes.c_void_p()
        _lib.check(self._lib.rgb_comm_init(ctypes.cast(uid, ctypes.c_void_p), self.world, self.rank, ctypes.byref(h)),
                   "comm_init")
        self.handle = h

    def allreduce_(self, flat: torch.Tensor) -> torch.Tensor:
        import ctypes

        from . import _lib
        _lib.check(self._lib.rgb_allreduce_grads(self.handle, ctypes.c_void_p(flat.data_ptr()), flat.numel(),
                                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return flat

    def max_(self, value: float, device=None) -> float:
        import ctypes

        from . import _lib
        if self.world == 1:
            return value
        t = torch.tensor([value], dtype=torch.float64, device=device or "cuda")
        _lib.check(self._lib.rgb_allreduce_f64(self.handle, ctypes.c_void_p(t.data_ptr()), 1, 1,
                                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return float(t.item())

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.rgb_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


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
