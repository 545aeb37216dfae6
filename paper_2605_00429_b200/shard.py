"""Query sharding rules for multi-GPU runs.

Queries are independent (REF/SPEC.md:518-519), so there is no exchange step: each GPU answers its
own rows against its own replica of the read-only structure.

  * device_shard   -- an even contiguous split of ONE batch (strong scaling); the same rule the C++
                      engine applies when one process drives several GPUs (p2m_engine.cu, p2m_query)
  * spatial_shard  -- strong scaling by Morton-range partitions of ONE batch: rank r owns the rows
                      whose coarse Morton key lies in its key range, the ranges cut so every rank gets
                      ~n/world rows.  Each GPU then sees a compact spatial region, so rows per site
                      and the L2 working set per GPU stay those of the single-GPU run (an even split
                      of c5's 100 M rows leaves ~6 rows per site per GPU at 8 GPUs)
  * rank_slice     -- weak scaling: rank r owns its own full batch [r*n, (r+1)*n) of the config's
                      counter-based query sequence
  * max_over_ranks -- the step time of a multi-GPU run is the max over ranks
"""
from __future__ import annotations

import numpy as np


def rank_slice(rank: int, world: int, n_per_rank: int):
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return rank * n_per_rank, n_per_rank


def device_shard(n: int, n_devices: int, k: int):
    if not (0 <= k < n_devices):
        raise ValueError("shard index out of range")
    b = n * k // n_devices
    e = n * (k + 1) // n_devices
    return b, e - b


def morton_box(points):
    """The key box of spatial_shard: 1.5x the points' AABB about its centre (as the device's
    Morton key box, p2m_engine.cu) -> (lo[3], extent[3])."""
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    lo, hi = p.min(0), p.max(0)
    c, h = (lo + hi) / 2, np.maximum((hi - lo) / 2, 1e-12) * 1.5
    return c - h, 2 * h


_SPREAD = None


def morton_keys(q, box, bits: int = 7):
    """Coarse Morton key (3*bits bits) of each row of q in box; rows outside the box clamp."""
    global _SPREAD
    if _SPREAD is None or len(_SPREAD) != (1 << bits):
        s = np.zeros(1 << bits, np.uint64)
        for i in range(1 << bits):
            v = 0
            for b in range(bits):
                v |= ((i >> b) & 1) << (3 * b)
            s[i] = v
        _SPREAD = s
    lo, ext = box
    g = np.floor((np.asarray(q, dtype=np.float64) - lo) / ext * (1 << bits))
    g = np.clip(g, 0, (1 << bits) - 1).astype(np.int64)
    return _SPREAD[g[:, 0]] | (_SPREAD[g[:, 1]] << np.uint64(1)) | (_SPREAD[g[:, 2]] << np.uint64(2))


def spatial_bounds(key_counts, world: int):
    """Key-range boundaries [b_0 = 0, ..., b_world = K) cutting the key histogram into world parts
    of ~equal row counts (whole key cells never split)."""
    cum = np.cumsum(key_counts)
    n = int(cum[-1]) if len(cum) else 0
    b = [0]
    for r in range(1, world):
        b.append(int(np.searchsorted(cum, n * r / world, side="left")) + 1)
    b.append(len(key_counts))
    return np.maximum.accumulate(np.array(b))


def spatial_shard(gen, n_total: int, world: int, rank: int, box, bits: int = 7, chunk: int = 1 << 23,
                  parts_per_rank: int = 1):
    """Rank `rank`'s rows of ONE batch under the Morton-range partition.  gen(first, count) yields rows
    [first, first+count) of the batch.  Two passes over the batch (key histogram, then selection);
    returns (q rows of this rank in batch order, their batch row indices).

    parts_per_rank = k > 1 cuts the key order into world*k ranges of ~equal row counts and deals them
    round-robin (rank r owns ranges r, r + world, ...): every range is still a compact region at the
    batch's full row density (rows per site as in the single-GPU run), but a rank's time now averages
    over k regions of the domain -- on c5 equal-row regions differ by up to 1.3x in scan time
    (DESIGN.md section 8), which one range per rank turns into load imbalance."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    if parts_per_rank < 1:
        raise ValueError("parts_per_rank must be >= 1")
    counts = np.zeros(1 << (3 * bits), np.int64)
    for a in range(0, n_total, chunk):
        k = morton_keys(gen(a, min(chunk, n_total - a)), box, bits)
        counts += np.bincount(k.astype(np.int64), minlength=len(counts))
    bnd = spatial_bounds(counts, world * parts_per_rank)
    qs, idx = [], []
    for a in range(0, n_total, chunk):
        q = gen(a, min(chunk, n_total - a))
        k = morton_keys(q, box, bits).astype(np.int64)
        part = np.searchsorted(bnd, k, side="right") - 1
        sel = np.flatnonzero(part % world == rank)
        qs.append(q[sel])
        idx.append(sel + a)
    if not qs:
        return np.zeros((0, 3)), np.zeros(0, np.int64)
    return np.concatenate(qs), np.concatenate(idx)


def max_over_ranks(value: float, dist=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
