"""torch.distributed bootstrap for the sharded path (one process per GPU).

torch.distributed is plumbing only: it broadcasts the 128-byte ncclUniqueId
that rank 0 obtains from libsv (sv_nccl_unique_id) and provides barriers and
the max-over-ranks reduction of timings.  All state-vector data moves through
libsv's own NCCL communicator (qubit-swap all-to-all, scalar allreduce).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

from . import _sv


def env_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process if unset)."""
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def init_process_group(backend: str | None = None) -> tuple[int, int, int]:
    rank, world, local = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string from `src` over the default process group."""
    obj = [payload]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def shared_nccl_id() -> bytes:
    """Rank 0 creates the libsv NCCL unique id; every rank returns the same bytes."""
    rank = dist.get_rank()
    payload = _sv.sv_nccl_unique_id() if rank == 0 else None
    return broadcast_bytes(payload, 0)


def max_over_ranks(value: float) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sharded_init(n: int, seed: int = 0, dtype: int = _sv.SV_C64, init: int = _sv.SV_INIT_UNIFORM,
                 stream: int | None = None) -> _sv.Ctx:
    """sv_init on every rank of the default process group (one GPU per rank)."""
    rank, world, local = env_world()
    if world == 1:
        return _sv.sv_init(n, seed, dtype, init, device=local, stream=stream)
    nid = shared_nccl_id()
    return _sv.sv_init(n, seed, dtype, init, rank=rank, world=world, nccl_id=nid, device=local, stream=stream)
