"""The N>1 path on CPU (gloo, world_size 2): bench.py's weak-scaling sharding (each rank owns the
contiguous slice [rank*n, (rank+1)*n) of the config's counter-based query sequence, builds its own
replica, and answers it with no data-path collective) reproduces the single-process answer over
[0, world*n), and the timing reduction is a max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import shard

N_PER_RANK = 3000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V, F = P.icosphere(3)
    h = P.HostEngine.build(V, F, P.BuildConfig(n_threads=2))
    first, count = shard.rank_slice(rank, world, N_PER_RANK)
    q = P.gen_queries(1, V, F, first, count)
    r = O.OracleEngine(h.arrays()).batch_query(q, threads=2)
    part = torch.from_numpy(np.concatenate([r["distance"], r["face"].astype(np.float64), r["site"].astype(np.float64)]))
    parts = [torch.zeros_like(part) for _ in range(world)]
    dist.all_gather(parts, part)
    t = shard.max_over_ranks(0.5 + rank, dist)  # each rank "took" 0.5 + rank seconds
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), torch.stack(parts).numpy())
        np.save(os.path.join(out_dir, "tmax.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_weak_scaling_matches_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "gathered.npy")
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 1.5
    V, F = P.icosphere(3)
    h = P.HostEngine.build(V, F)
    q = P.gen_queries(1, V, F, 0, world * N_PER_RANK)
    r = O.OracleEngine(h.arrays()).batch_query(q)
    for rank in range(world):
        sl = slice(rank * N_PER_RANK, (rank + 1) * N_PER_RANK)
        n = N_PER_RANK
        assert got[rank][:n].tobytes() == r["distance"][sl].tobytes()
        assert np.array_equal(got[rank][n:2 * n].astype(np.uint32), r["face"][sl])
        assert np.array_equal(got[rank][2 * n:].astype(np.uint32), r["site"][sl])


def test_rank_slices_partition():
    n = 1000
    sl = [shard.rank_slice(r, 4, n) for r in range(4)]
    assert sl == [(0, n), (n, n), (2 * n, n), (3 * n, n)]
    # even split of one batch over devices (p2m_query's host-side sharding rule)
    for total in (0, 1, 7, 1000, 1001):
        for g in (1, 2, 3, 8):
            b = [shard.device_shard(total, g, k) for k in range(g)]
            assert sum(c for _, c in b) == total
            assert all(b[k][0] + b[k][1] == b[k + 1][0] for k in range(g - 1))
            assert max(c for _, c in b) - min(c for _, c in b) <= 1
