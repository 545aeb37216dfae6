"""GPU parity: the CUDA query path (through the C ABI) vs the CPU oracle on identical inputs.

Bar (BASELINE.json north_star): site and face ids exact, distance and closest point within 1e-6
relative.  fp64 with --fmad=false and the reference's operation order makes every row
bit-identical, which is what these tests assert (tolerance 0, stricter than 1e-6 relative).
Edge cases follow the SPEC's examples: empty batch (REF/SPEC.md:503), duplicated point (504),
q = mesh vertex (494), out-of-domain rows answered by the fallback (491, 611), tiny meshes."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from conftest import big_config, oracle_checker
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L

pytestmark = pytest.mark.gpu

TET_V = np.array([[1.0, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]])
TET_F = np.array([[0, 1, 2], [0, 3, 1], [0, 2, 3], [1, 3, 2]], np.uint32)


def _compare(r, ref, n):
    for k in ("site", "face", "flags"):
        a, b = getattr(r, k), ref[k]
        bad = np.flatnonzero(a != b)
        assert len(bad) == 0, f"{k}: {len(bad)} of {n} rows differ, first {bad[:5]}"
    for k in ("distance", "closest"):
        a, b = getattr(r, k), ref[k]
        assert a.tobytes() == b.tobytes(), f"{k} not bit-identical"


def _check_counters(r, ref, sequential):
    c, rc = r.counters, ref["counters"]
    # candidates (= list length of the nearest site, REF/SPEC.md:511) are deterministic
    assert c["candidates_visited"] == rc["candidates_visited"]
    assert c["fallbacks"] == rc["fallbacks"]
    assert c["exact_evaluations"] + c["pruned"] == c["candidates_visited"]  # REF/SPEC.md:511
    if sequential:
        # the fused per-row path walks the k-d tree and the list in the oracle's order: all match
        assert c["exact_evaluations"] == rc["exact_evaluations"]
        assert c["kd_nodes_visited"] == rc["kd_nodes_visited"]
    else:
        # the grouped path locates sites through the exact grid: it counts grid candidates
        assert c["kd_nodes_visited"] >= c["n_queries"]


@pytest.mark.parametrize("fixture,nq,cfg", [("ico3", 20000, None), ("c1", 300000, 1), ("c2", 300000, 2)])
def test_parity_vs_oracle(request, fixture, nq, cfg):
    V, F, h = request.getfixturevalue(fixture)
    if cfg is None:
        q = np.random.default_rng(3).uniform(-1.3, 1.3, size=(nq, 3))
    else:
        q = P.gen_queries(cfg, V, F, 0, nq)
    eng = P.Engine(h)
    r = eng.batch_query(q)
    ref = oracle_checker(h.arrays()).batch_query(q, prune=O.PRUNE_SAFE)
    _compare(r, ref, nq)
    _check_counters(r, ref, sequential=False)


@pytest.mark.parametrize("mode", [0, 1])
def test_scan_modes_identical(c2, mode):
    """Grouped (site tiles, shared memory) and fused (one thread per row) scans give the same rows."""
    V, F, h = c2
    q = P.gen_queries(2, V, F, 500_000, 100_000)
    eng = P.Engine(h)
    L.check(L.cuda().p2m_set_scan_mode(eng.handle, mode))
    r = eng.batch_query(q)
    ref = oracle_checker(h.arrays()).batch_query(q, prune=O.PRUNE_SAFE)
    _compare(r, ref, len(q))
    _check_counters(r, ref, sequential=(mode == 1))


def test_golden_engine_on_gpu():
    """The committed reference-generated fixture (tests/golden/engine_ico2.npz) on the GPU."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "engine_ico2.npz"))
    h = P.HostEngine.build(g["vertices"], g["faces"])
    a = h.arrays()
    assert a["list_faces"].tobytes() == g["list_faces"].tobytes()  # same build on this box
    r = P.Engine(h).batch_query(g["q"])
    for k in ("distance", "closest", "face", "site", "flags"):
        assert getattr(r, k).tobytes() == g[k].tobytes(), k


def test_empty_and_duplicated_batches(ico3):
    V, F, h = ico3
    eng = P.Engine(h)
    r = eng.batch_query(np.zeros((0, 3)))
    assert len(r.distance) == 0 and all(v == 0 for v in r.counters.values())  # REF/SPEC.md:503
    for mode in (0, 1):
        L.check(L.cuda().p2m_set_scan_mode(eng.handle, mode))
        one = eng.batch_query(np.array([[0.3, -0.2, 0.5]]))
        many = eng.batch_query(np.tile([[0.3, -0.2, 0.5]], (1000, 1)))
        assert np.all(many.distance == one.distance[0]) and np.all(many.face == one.face[0])
        # REF/SPEC.md:504; exact evaluations depend on how the grouped scan splits a tile (a lone row
        # gets 8 replicas), so that counter is checked on the sequential fused path only
        keys = ("candidates_visited", "kd_nodes_visited") + (("exact_evaluations",) if mode == 1 else ())
        for k in keys:
            assert many.counters[k] == 1000 * one.counters[k], (mode, k)


def test_vertex_queries_and_out_of_domain(ico3):
    V, F, h = ico3
    eng = P.Engine(h)
    r = eng.batch_query(V)
    assert np.all(r.distance == 0.0)  # REF/SPEC.md:494
    for i in range(0, len(V), 17):
        assert i in F[r.face[i]]
    a = h.arrays()
    far = np.array([[100.0, 0, 0], [0, -250.0, 3.0], [1e6, 1e6, 1e6], [a["domain"][3] + 1e-9, 0, 0]])
    r = eng.batch_query(far)
    assert np.all((r.flags & 3) == 3) and r.counters["fallbacks"] == len(far)
    tri = a["tri"].reshape(-1, 9)
    for i, q in enumerate(far):
        d2, p, f = O.brute_force_closest(tri, q)
        assert r.face[i] == f and r.distance[i] == np.sqrt(d2) and r.closest[i].tobytes() == p.tobytes()


@pytest.mark.parametrize("mesh", ["tri", "tet"])
def test_tiny_meshes(mesh):
    V, F = {"tri": (np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]]), np.array([[0, 1, 2]], np.uint32)),
            "tet": (TET_V, TET_F)}[mesh]
    h = P.HostEngine.build(V, F)
    q = np.random.default_rng(1).uniform(-3, 3, size=(5000, 3))
    r = P.Engine(h).batch_query(q)
    ref = oracle_checker(h.arrays()).batch_query(q)
    _compare(r, ref, len(q))


def test_nearest_site_and_per_query_counters(c1):
    import torch
    V, F, h = c1
    q = P.gen_queries(1, V, F, 0, 50_000)
    eng = P.Engine(h)
    dq = torch.from_numpy(q).cuda()
    site = torch.empty(len(q), dtype=torch.int32, device="cuda")
    pq = torch.empty((len(q), 3), dtype=torch.int64, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    L.check(L.cuda().p2m_nearest_site_device(eng.handle, 0, C.c_void_p(dq.data_ptr()), len(q),
                                             C.c_void_p(site.data_ptr()), s))
    L.check(L.cuda().p2m_set_scan_mode(eng.handle, 1))  # oracle-ordered path: node counts comparable
    L.check(L.cuda().p2m_query_device_counters(eng.handle, 0, C.c_void_p(dq.data_ptr()), len(q),
                                               C.c_void_p(pq.data_ptr()), s))
    torch.cuda.synchronize()
    ref = oracle_checker(h.arrays()).batch_query(q, per_query=True)
    assert np.array_equal(site.cpu().numpy().astype(np.uint32), ref["site"])
    pq = pq.cpu().numpy()
    assert np.array_equal(pq[:, 0], ref["per_query"][:, 0])
    assert np.array_equal(pq[:, 2], ref["per_query"][:, 2])


def test_multi_slot_engine_shards_and_replicates(c2):
    """Two replicas on device 0 exercise the peer-replica copy and the per-device host threads of
    p2m_query on a single GPU; rows must not depend on the shard they land in."""
    V, F, h = c2
    q = P.gen_queries(2, V, F, 0, 200_001)
    r1 = P.Engine(h, devices=[0]).batch_query(q)
    e2 = P.Engine(h, devices=[0, 0])
    assert e2.info()["n_devices"] == 2
    r2 = e2.batch_query(q)
    for k in ("distance", "closest", "face", "site", "flags"):
        assert getattr(r1, k).tobytes() == getattr(r2, k).tobytes(), k
    assert r1.counters["candidates_visited"] == r2.counters["candidates_visited"]


def test_device_api_on_torch_stream(c2):
    """p2m_query_device on caller-owned device buffers and stream == the host-buffer API."""
    import torch
    V, F, h = c2
    q = P.gen_queries(2, V, F, 7, 123_457)
    eng = P.Engine(h)
    n = len(q)
    dq = torch.from_numpy(q).cuda()
    outs = [torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda")] + \
           [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(3)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        L.check(L.cuda().p2m_query_device(eng.handle, 0, C.c_void_p(dq.data_ptr()), n,
                                          *[C.c_void_p(t.data_ptr()) for t in outs],
                                          C.c_void_p(st.cuda_stream), None))
    st.synchronize()
    r = eng.batch_query(q)
    assert outs[0].cpu().numpy().tobytes() == r.distance.tobytes()
    assert np.array_equal(outs[2].cpu().numpy().astype(np.uint32), r.face)


def test_kernel_launch_count(ico3):
    V, F, h = ico3
    eng = P.Engine(h)
    n = C.c_int()
    L.check(L.cuda().p2m_kernels_per_query(eng.handle, 100000, C.byref(n)))
    assert 6 <= n.value <= 30


@pytest.mark.slow
@pytest.mark.parametrize("cfg,nq", [(3, 1_000_000), (4, 1_000_000), (5, 2_000_000)])
def test_parity_large_configs(cfg, nq):
    """c3..c5 through the public host API, every row bit-identical to the reference CPU query path
    (oracle/_ref) -- 2 M rows on c5, the benchmark config."""
    V, F, h = big_config(cfg)
    q = P.gen_queries(cfg, V, F, 0, nq)
    r = P.Engine(h).batch_query(q)
    ref = oracle_checker(h.arrays()).batch_query(q, prune=O.PRUNE_SAFE)
    _compare(r, ref, len(q))
    _check_counters(r, ref, sequential=False)


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_exact_vs_brute_force(cfg, c2):
    """Acceptance (REF/SPEC.md:508, 665-667): on a 10^4-query sample of each benchmark config the
    GPU answer equals brute_force_closest over ALL faces (REF/SPEC.md:536-544) -- the check that
    does not trust the interception tables at all.  Distance and closest point bit-identical; the
    face id may differ only on an exact tie of d^2 (never observed: the tables keep every tie)."""
    V, F, h = c2 if cfg == 2 else big_config(cfg)
    q = P.gen_queries(cfg, V, F, 3_000_000, 10_000)
    r = P.Engine(h).batch_query(q)
    tri = h.arrays()["tri"].reshape(-1, 9)
    bf = O.batch_brute_force(tri, q, reference=O.have_reference())
    same_face = r.face == bf["face"]
    d2 = r.distance * r.distance
    assert r.distance.tobytes() == np.sqrt(bf["d2"]).tobytes()
    assert np.all(same_face | (bf["d2"] == d2)), f"{(~same_face).sum()} rows differ"
    assert r.closest[same_face].tobytes() == bf["closest"][same_face].tobytes()
    assert (~same_face).sum() == 0


def test_grid_and_kdtree_locate_agree(c2):
    """The exact grid cell-locate and the k-d tree give identical nearest sites (and rows), including
    rows outside the grid box (k-d tree fallback inside k_descend)."""
    import os
    V, F, h = c2
    q = np.concatenate([P.gen_queries(2, V, F, 3_000_000, 200_000),
                        np.random.default_rng(9).uniform(-4, 4, size=(20_000, 3))])
    r_grid = P.Engine(h).batch_query(q)
    os.environ["P2M_NO_GRID"] = "1"
    try:
        r_kd = P.Engine(h).batch_query(q)
    finally:
        del os.environ["P2M_NO_GRID"]
    for k in ("distance", "closest", "face", "site", "flags"):
        assert getattr(r_grid, k).tobytes() == getattr(r_kd, k).tobytes(), k
    ref = oracle_checker(h.arrays()).batch_query(q)
    _compare(r_grid, ref, len(q))


def _surface_probes(V, F, n, rng, scales):
    """Points on faces, at vertices and on edges, pushed off the surface by tiny normal offsets --
    the regime where the fp32 pre-filters run closest to their margins."""
    t = F[rng.integers(0, len(F), n)]
    a, b, c = V[t[:, 0]], V[t[:, 1]], V[t[:, 2]]
    w = rng.dirichlet([1, 1, 1], size=n)
    kind = rng.integers(0, 3, n)
    w[kind == 1] = [1.0, 0.0, 0.0]                      # vertices
    w[kind == 2] = np.c_[rng.uniform(size=(kind == 2).sum()), np.zeros(((kind == 2).sum(), 1)), np.zeros(((kind == 2).sum(), 1))]
    w[kind == 2, 1] = 1.0 - w[kind == 2, 0]             # edges ab
    p = w[:, :1] * a + w[:, 1:2] * b + w[:, 2:3] * c
    nrm = np.cross(b - a, c - a)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    off = rng.choice(scales, size=n) * rng.choice([-1.0, 1.0], size=n)
    return p + nrm * off[:, None]


@pytest.mark.parametrize("variant", ["far_translated", "slivers"])
def test_fp32_prefilters_stress(variant):
    rng = np.random.default_rng(17)
    V, F = P.icosphere(3)
    if variant == "far_translated":
        V = V * 1e3 + np.array([5e3, -2e3, 1e3])       # large |coordinates| vs feature size
        scale = 1e3
    else:
        V = V * (1.0 + 0.15 * rng.standard_normal((len(V), 1)))  # bumpy: thin and obtuse faces
        V[::7] += 0.02 * rng.standard_normal((len(V[::7]), 3))
        scale = 1.0
    h = P.HostEngine.build(V, F)
    Vv, Ff = h.mesh()
    q = np.concatenate([
        _surface_probes(Vv, Ff, 60_000, rng, np.array([0.0, 1e-12, 1e-9, 1e-6, 1e-4, 1e-2]) * scale),
        Vv.mean(0) + rng.uniform(-1.3, 1.3, size=(40_000, 3)) * scale,
    ])
    r = P.Engine(h).batch_query(q)
    ref = oracle_checker(h.arrays()).batch_query(q)
    _compare(r, ref, len(q))


@pytest.mark.parametrize("chunks", ["0", "1", "3", "7"])
def test_host_api_chunk_schedules_identical(c2, chunks, monkeypatch):
    """p2m_query pipelines host-buffer batches in chunks (geometric by default, P2M_E2E_CHUNKS=k
    equal chunks); rows never depend on the chunking and equal the device-resident path."""
    import torch
    V, F, h = c2
    q = P.gen_queries(2, V, F, 1_000_000, 700_000)
    monkeypatch.setenv("P2M_E2E_CHUNKS", chunks)
    r = P.Engine(h).batch_query(q)
    monkeypatch.delenv("P2M_E2E_CHUNKS")
    eng = P.Engine(h)
    n = len(q)
    dq = torch.from_numpy(q).cuda()
    od = torch.empty(n, dtype=torch.float64, device="cuda")
    oc = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    of, osi, ofl = (torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(3))
    vp = lambda t: C.c_void_p(t.data_ptr())
    L.check(L.cuda().p2m_query_device(eng.handle, 0, vp(dq), n, vp(od), vp(oc), vp(of), vp(osi), vp(ofl),
                                      None, None))
    torch.cuda.synchronize()
    assert r.distance.tobytes() == od.cpu().numpy().tobytes()
    assert r.closest.tobytes() == oc.cpu().numpy().tobytes()
    assert np.array_equal(r.face, of.cpu().numpy().view(np.uint32))
    assert np.array_equal(r.site, osi.cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("env", [
    {"P2M_SMALL_CHUNKS": "0"},                 # every tile on the CTA path
    {"P2M_SMALL_CHUNKS": "4"},                 # more tiles one warp per tile (side-stream kernel)
    {"P2M_TILE_ORDER": "0"}, {"P2M_TILE_ORDER": "1"}, {"P2M_TILE_ORDER": "2"},  # launch orders
    {"P2M_MORTON_BITS": "30"}, {"P2M_MORTON_BITS": "9"},  # finer / much coarser Morton order
    {"P2M_LONG_TILE": "128"},                  # heavy-site tile height
    {"P2M_HEAVY_E": "16"},                     # many more heavy sites (short tiles)
    {"P2M_NO_SEED": "1"}, {"P2M_NO_BATCH": "1"},  # without the d_min seeds / group-sphere levels
    {"P2M_NO_DEEP_SEED": "1"},                 # group-point seeds only (no per-row exact seed face)
    {"P2M_NO_WARP_QUEUE": "1"},                # warp tiles evaluate batch by batch (union walk), no pair queue
    {"P2M_NO_WARP_QUEUE": "1", "P2M_SCAN_WARP": "1"},
    {"P2M_DENSE_PAIRS": "1"}, {"P2M_DENSE_PAIRS": "1000"},  # warp tiles: every batch walks the union / queues its pairs
    {"P2M_NO_TVOTE": "1"},                     # chunk / batch votes by broadcast per group (not transposed)
    {"P2M_NO_TVOTE": "1", "P2M_SCAN_WARP": "1"},
    {"P2M_NO_SPATIAL": "1"},                   # lists scanned in ascending face order
    {"P2M_SCAN_WARP": "1"},                    # every tile a 32-row warp tile (no CTA tiles)
    {"P2M_WARP_MIN_CHUNKS": "0"},              # no warp tiles beyond the small-list ones
    {"P2M_WARP_MIN_CHUNKS": "3"},              # warp tiles only for lists of >= 3 chunks
    {"P2M_SMALL_CHUNKS": "0", "P2M_WARP_MIN_CHUNKS": "1"},  # warp tiles without small-list tiles
])
def test_scan_schedules_identical(c2, env, monkeypatch):
    """The tile partition (CTA tiles vs one-warp small tiles), their launch order, the Morton
    granularity and the heavy-tile height change which warps scan what and in which order -- never
    the rows: every schedule equals the default one and the oracle bit for bit.  400 k rows leave
    ~23 rows per site, so small tiles dominate."""
    V, F, h = c2
    q = P.gen_queries(2, V, F, 2_000_000, 400_000)
    base = P.Engine(h).batch_query(q)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    r = P.Engine(h).batch_query(q)
    ref = {"site": base.site, "face": base.face, "flags": base.flags, "distance": base.distance,
           "closest": base.closest}
    _compare(r, ref, len(q))
    if env == {"P2M_SMALL_CHUNKS": "4"}:
        _compare(r, oracle_checker(h.arrays()).batch_query(q, prune=O.PRUNE_SAFE), len(q))


def test_concurrent_device_calls_one_engine(c2):
    """One engine queried from several host threads at once, each on its own stream
    (REF/SPEC.md:518-519: queries are pure and concurrent): the fork/join of the small-tile side
    stream must not interleave between calls.  Every thread's rows equal the serial answer."""
    import threading
    import torch
    V, F, h = c2
    eng = P.Engine(h)
    qs = [P.gen_queries(2, V, F, 3_000_000 + 200_000 * k, 150_000) for k in range(4)]
    want = [eng.batch_query(q) for q in qs]
    lib = L.cuda()
    vp = lambda t: C.c_void_p(t.data_ptr())
    errs = []

    def worker(k):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            n = len(qs[k])
            dq = torch.from_numpy(qs[k]).cuda()
            for _ in range(5):
                od = torch.empty(n, dtype=torch.float64, device="cuda")
                of, osi, ofl = (torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(3))
                oc = torch.empty((n, 3), dtype=torch.float64, device="cuda")
                torch.cuda.current_stream().synchronize()
                L.check(lib.p2m_query_device(eng.handle, 0, vp(dq), n, vp(od), vp(oc), vp(of), vp(osi), vp(ofl),
                                             C.c_void_p(st.cuda_stream), None))
                st.synchronize()
                assert od.cpu().numpy().tobytes() == want[k].distance.tobytes()
                assert np.array_equal(of.cpu().numpy().view(np.uint32), want[k].face)
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


@pytest.mark.parametrize("sched", ["0.05,3,0.4,0.1", "0.3,1,0.3,0.05"])
def test_host_api_geometric_schedules_identical(c2, sched, monkeypatch):
    """The geometric host-API schedule (first, growth, cap, tail) never changes a row."""
    V, F, h = c2
    q = P.gen_queries(2, V, F, 1_500_000, 900_000)
    base = P.Engine(h).batch_query(q)
    monkeypatch.setenv("P2M_E2E_SCHED", sched)
    r = P.Engine(h).batch_query(q)
    _compare(r, {"site": base.site, "face": base.face, "flags": base.flags, "distance": base.distance,
                 "closest": base.closest}, len(q))


@pytest.mark.parametrize("chunks,with_flags", [("0", True), ("2", False)])
def test_host_api_pageable_equals_pinned(c2, chunks, with_flags, monkeypatch):
    """p2m_query on pageable caller arrays runs through pinned bounce rings (1 M-row sub-chunks,
    packed/unpacked by host threads); on page-locked arrays the DMA engines read and write them
    directly.  Both give the same rows, bit for bit, across several sub-chunks per chunk, with and
    without the optional flags array."""
    import torch
    V, F, h = c2
    q = P.gen_queries(2, V, F, 4_000_000, 2_600_000)
    n = len(q)
    monkeypatch.setenv("P2M_E2E_CHUNKS", chunks)
    eng = P.Engine(h)
    lib = L.cuda()
    pd, pc = np.full(n, -1.0), np.full((n, 3), -1.0)
    pf, ps, pfl = (np.zeros(n, np.uint32) for _ in range(3))
    L.check(lib.p2m_query(eng.handle, L.ptr(q), n, L.ptr(pd), L.ptr(pc), L.ptr(pf, L.u32p), L.ptr(ps, L.u32p),
                          L.ptr(pfl, L.u32p) if with_flags else None, None))
    qp = torch.from_numpy(q).pin_memory()
    od = torch.empty(n, dtype=torch.float64).pin_memory()
    oc = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    of, osi, ofl = (torch.zeros(n, dtype=torch.int32).pin_memory() for _ in range(3))
    dp = lambda t: C.cast(C.c_void_p(t.data_ptr()), L.dp)
    up = lambda t: C.cast(C.c_void_p(t.data_ptr()), L.u32p)
    L.check(lib.p2m_query(eng.handle, dp(qp), n, dp(od), dp(oc), up(of), up(osi), up(ofl) if with_flags else None, None))
    assert pd.tobytes() == od.numpy().tobytes()
    assert pc.tobytes() == oc.numpy().tobytes()
    assert np.array_equal(pf, of.numpy().view(np.uint32))
    assert np.array_equal(ps, osi.numpy().view(np.uint32))
    if with_flags:
        assert np.array_equal(pfl, ofl.numpy().view(np.uint32))


def test_table_miss_falls_back_exactly(ico3):
    """A caller-filled desc whose list for site 0 is NOT a superset (one far face only): the grouped
    scan's d_min seed |q - v| prunes that face, the row would keep no face at all -- it is answered by
    the exact BVH fallback instead and flagged FALLBACK | TABLE_MISS (the seed assumes the
    Theorem-1 superset invariant, REF/SPEC.md:435).  Rows of every other site are unchanged."""
    V, F, h = ico3
    a = h.arrays()
    off = a["list_offsets"].astype(np.uint64)
    lf = a["list_faces"].astype(np.uint32)
    tri = a["tri"].reshape(-1, 9)
    cen = tri.reshape(-1, 3, 3).mean(1)
    far = int(np.argmax(np.linalg.norm(cen - V[0], axis=1)))
    new_lf = np.concatenate([lf[: off[0]], np.array([far], np.uint32), lf[off[1]:]])
    new_off = off.copy()
    new_off[1:] = off[1:] - (off[1] - off[0]) + 1
    d = h.desc()
    d.list_offsets = new_off.ctypes.data_as(L.u64p)
    d.list_faces = new_lf.ctypes.data_as(L.u32p)
    eng = P.Engine.from_desc(d, keep=(new_off, new_lf))
    rng = np.random.default_rng(11)
    q = np.concatenate([V[0] * 1.02 + rng.normal(0, 0.01, size=(3000, 3)),
                        rng.uniform(-1.3, 1.3, size=(3000, 3))])
    r = eng.batch_query(q)
    base = P.Engine(h).batch_query(q)
    hit = r.site == 0
    assert hit.sum() > 100
    assert np.all((r.flags[hit] & 5) == 5) and np.all((r.flags[~hit] & 4) == 0)
    for i in np.flatnonzero(hit)[:300]:
        d2, p, f = O.brute_force_closest(tri, q[i])
        assert r.face[i] == f and r.distance[i] == np.sqrt(d2) and r.closest[i].tobytes() == p.tobytes()
    # the fallback answer is the exact one, so it equals the superset engine's row
    assert r.distance.tobytes() == base.distance.tobytes() and np.array_equal(r.face, base.face)
    assert np.array_equal(r.flags[~hit], base.flags[~hit])


def test_device_image_round_trip(c2, tmp_path):
    """the engine saved as its packed device layout and loaded straight into
    it (no host engine, no re-packing) answers bit-identically to the oracle and to the engine that
    was saved (REF/SPEC.md:588-591: round trip gives identical query results); corrupt and truncated
    files fail with P2M_ERR_IO before anything reaches the device."""
    V, F, h = c2
    q = P.gen_queries(2, V, F, 5_000_000, 300_000)
    eng = P.Engine(h)
    path = str(tmp_path / "c2.p2md")
    eng.save(path)
    loaded = P.Engine.load(path)
    r0, r1 = eng.batch_query(q), loaded.batch_query(q)
    for k in ("distance", "closest", "face", "site", "flags"):
        assert getattr(r0, k).tobytes() == getattr(r1, k).tobytes(), k
    _compare(r1, oracle_checker(h.arrays()).batch_query(q, prune=O.PRUNE_SAFE), len(q))
    assert loaded.info()["device_bytes"] == eng.info()["device_bytes"]
    blob = open(path, "rb").read()
    for name, data in (("trunc", blob[: len(blob) // 2]), ("flip", blob[:200] + bytes([blob[200] ^ 1]) + blob[201:]),
                       ("magic", b"XXXX" + blob[4:])):
        bad = str(tmp_path / f"{name}.p2md")
        open(bad, "wb").write(data)
        with pytest.raises(L.P2MError) as ei:
            P.Engine.load(bad)
        assert ei.value.code == -6, name
    # replicated on two slots from the image (same GPU twice: the peer-copy path)
    two = P.Engine.load(path, devices=[0, 0])
    r2 = two.batch_query(q)
    assert r2.distance.tobytes() == r0.distance.tobytes() and np.array_equal(r2.face, r0.face)


def test_device_built_grid_without_cell_boxes(c2):
    """An external builder's desc without Voronoi cell boxes (site_cell_box = NULL): the engine
    builds the exact cell-locate grid on the device from the sites alone (p2m_grid.cu) instead of
    falling back to the per-thread k-d descent.  Rows are bit-identical to the box-built grid and to
    the oracle; the descent time is reported against the box-built grid."""
    import torch
    V, F, h = c2
    d = h.desc()
    d.site_cell_box = None
    eng_dev = P.Engine.from_desc(d)
    eng_box = P.Engine(h)
    q = P.gen_queries(2, V, F, 0, 2_000_000)
    a, b = eng_dev.batch_query(q), eng_box.batch_query(q)
    for k in ("distance", "closest", "face", "site", "flags"):
        assert getattr(a, k).tobytes() == getattr(b, k).tobytes(), k
    ref = oracle_checker(h.arrays()).batch_query(q[:300_000], prune=O.PRUNE_SAFE)
    for k in ("site", "face"):
        assert np.array_equal(getattr(a, k)[:300_000], ref[k]), k
    assert a.distance[:300_000].tobytes() == ref["distance"].tobytes()
    # grid candidates per query (kd_nodes_visited counts them): same order of magnitude
    assert a.counters["kd_nodes_visited"] <= 4 * b.counters["kd_nodes_visited"]
    n = len(q)
    dq = torch.from_numpy(q).cuda()
    outs = [torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, 3), dtype=torch.float64, device="cuda")] + \
           [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(3)]
    vp = lambda t: C.c_void_p(t.data_ptr())
    lib = L.cuda()
    t = {}
    for name, e in (("device_grid", eng_dev), ("box_grid", eng_box)):
        for _ in range(2):
            L.check(lib.p2m_query_device(e.handle, 0, vp(dq), n, *[vp(x) for x in outs], None, None))
        L.check(lib.p2m_set_profiling(e.handle, 1))
        for _ in range(5):
            L.check(lib.p2m_query_device(e.handle, 0, vp(dq), n, *[vp(x) for x in outs], None, None))
        torch.cuda.synchronize()
        ms = (C.c_float * 6)()
        L.check(lib.p2m_last_timings(e.handle, 0, ms))
        L.check(lib.p2m_set_profiling(e.handle, 0))
        t[name] = ms[2]
    print(f"descent ms: device-built grid {t['device_grid']:.3f}, box grid {t['box_grid']:.3f}")
    assert t["device_grid"] <= 3.0 * t["box_grid"]
