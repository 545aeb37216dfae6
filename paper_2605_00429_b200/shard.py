"""Query sharding rules for multi-GPU runs.

Queries are independent (REF/SPEC.md:518-519), so there is no exchange step: each GPU answers its
own rows against its own replica of the read-only structure.

  * rank_slice   -- one process per GPU (torchrun): weak scaling, rank r owns the contiguous slice
                    [r*n, (r+1)*n) of the config's counter-based query sequence
  * device_shard -- one process driving several GPUs (p2m_query): an even contiguous split of one
                    batch, the same rule the C++ engine applies (p2m_engine.cu, p2m_query)
  * max_over_ranks -- the step time of a multi-GPU run is the max over ranks
"""
from __future__ import annotations


def rank_slice(rank: int, world: int, n_per_rank: int):
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return rank * n_per_rank, n_per_rank


def device_shard(n: int, n_devices: int, k: int):
    b = n * k // n_devices
    e = n * (k + 1) // n_devices
    return b, e - b


def max_over_ranks(value: float, dist=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
