"""The N>1 path on CPU (gloo, world_size 2).  bench.py shards ONE batch over the ranks (strong
scaling, the metric's "100M queries sharded across 1/2/4/8 GPUs"): an even contiguous split or a
Morton-range spatial partition; each rank answers its own rows against its own copy of the engine
(rank 0 builds and saves the EngineIndexFile, rank 1 loads it) with no data-path collective.  The
union of the ranks' rows must reproduce the single-process answer row for row, and the timing
reduction is a max over ranks.  The weak-scaling rule (rank_slice) is checked the same way."""
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

N_TOTAL = 6000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V, F = P.icosphere(3)
    path = os.path.join(out_dir, "engine.p2mx")
    if rank == 0:                               # build once, the other rank loads the index file
        h = P.HostEngine.build(V, F, P.BuildConfig(n_threads=2))
        h.save(path)
    dist.barrier()
    if rank != 0:
        h = P.HostEngine.load(path, V, F)
    gen = lambda a, b: P.gen_queries(1, V, F, a, b)  # noqa: E731
    if mode == "even":
        first, count = shard.device_shard(N_TOTAL, world, rank)
        q, idx = gen(first, count), np.arange(first, first + count)
    elif mode == "spatial":
        A = h.arrays()
        box = shard.morton_box(A["site_xyz"][A["site_kind"] != 1])
        q, idx = shard.spatial_shard(gen, N_TOTAL, world, rank, box, bits=4, chunk=1000)
    else:                                       # weak: every rank its own N_TOTAL / world rows
        first, count = shard.rank_slice(rank, world, N_TOTAL // world)
        q, idx = gen(first, count), np.arange(first, first + count)
    r = O.OracleEngine(h.arrays()).batch_query(q, threads=2)
    rec = np.zeros((len(q), 4))
    rec[:, 0] = idx
    rec[:, 1] = r["distance"]
    rec[:, 2] = r["face"]
    rec[:, 3] = r["site"]
    n_loc = torch.tensor([len(q)])
    ns = [torch.zeros_like(n_loc) for _ in range(world)]
    dist.all_gather(ns, n_loc)
    m = int(max(int(x) for x in ns))
    pad = torch.full((m, 4), -1.0, dtype=torch.float64)
    pad[: len(q)] = torch.from_numpy(rec)
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    t = shard.max_over_ranks(0.5 + rank, dist)  # each rank "took" 0.5 + rank seconds
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), torch.cat(parts).numpy())
        np.save(os.path.join(out_dir, "counts.npy"), np.array([int(x) for x in ns]))
        np.save(os.path.join(out_dir, "tmax.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("mode", ["even", "spatial", "weak"])
def test_two_rank_sharding_matches_single_process(tmp_path, mode):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), mode), nprocs=world, join=True)
    got = np.load(tmp_path / "gathered.npy")
    got = got[got[:, 0] >= 0]
    counts = np.load(tmp_path / "counts.npy")
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 1.5
    assert counts.sum() == N_TOTAL
    if mode == "spatial":                        # balanced within the key-cell granularity
        assert counts.min() > 0.25 * N_TOTAL
    idx = got[:, 0].astype(np.int64)
    assert np.array_equal(np.sort(idx), np.arange(N_TOTAL))  # a partition of the batch
    V, F = P.icosphere(3)
    h = P.HostEngine.build(V, F)
    q = P.gen_queries(1, V, F, 0, N_TOTAL)
    r = O.OracleEngine(h.arrays()).batch_query(q)
    assert got[:, 1].tobytes() == r["distance"][idx].tobytes()
    assert np.array_equal(got[:, 2].astype(np.uint32), r["face"][idx])
    assert np.array_equal(got[:, 3].astype(np.uint32), r["site"][idx])


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


def test_spatial_partition_is_a_partition():
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1, 1, size=(20000, 3))
    gen = lambda a, b: pts[a:a + b]  # noqa: E731
    box = shard.morton_box(pts)
    for world in (1, 2, 3, 8):
        seen = []
        for r in range(world):
            q, idx = shard.spatial_shard(gen, len(pts), world, r, box, bits=5, chunk=3000)
            assert np.array_equal(q, pts[idx])
            assert np.all(np.diff(idx) > 0)           # batch order kept inside a part
            seen.append(idx)
            assert len(idx) > 0.5 * len(pts) / world  # balanced up to key-cell granularity
        allidx = np.concatenate(seen)
        assert np.array_equal(np.sort(allidx), np.arange(len(pts)))
        # several interleaved key ranges per rank (load balance): still a partition, still balanced,
        # and every rank's rows are the union of whole key ranges dealt round-robin
        seen = [shard.spatial_shard(gen, len(pts), world, r, box, bits=5, chunk=3000, parts_per_rank=4)[1]
                for r in range(world)]
        assert np.array_equal(np.sort(np.concatenate(seen)), np.arange(len(pts)))
        assert all(len(i) > 0.5 * len(pts) / world for i in seen)
        if world > 1:
            k5 = shard.morton_keys(pts, box, 5).astype(np.int64)
            bnd = shard.spatial_bounds(np.bincount(k5, minlength=1 << 15), world * 4)
            part = np.searchsorted(bnd, k5, side="right") - 1
            for r in range(world):
                assert np.array_equal(np.unique(part[seen[r]]) % world, np.full(len(np.unique(part[seen[r]])), r))
    # the key ranges are contiguous: every key of part r is below every key of part r+1
    k = shard.morton_keys(pts, box, 5)
    q0, i0 = shard.spatial_shard(gen, len(pts), 2, 0, box, bits=5)
    q1, i1 = shard.spatial_shard(gen, len(pts), 2, 1, box, bits=5)
    assert k[i0].max() < k[i1].min()
