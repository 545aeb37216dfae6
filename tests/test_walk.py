"""DelaunayWalk nearest_site (REF/SPEC.md:473-481, 516) and strategy
neutrality (REF/SPEC.md:510): KdTree and DelaunayWalk give identical nearest ids, and the device
engine's three strategies (grid, k-d tree, walk) give bit-identical QueryResults."""
import numpy as np
import pytest

import oracle as O
from conftest import oracle_checker
import paper_2605_00429_b200 as P


def _check_adjacency(off, adj, n):
    assert off[0] == 0 and len(off) == n + 1 and off[-1] == len(adj)
    pairs = set()
    for s in range(n):
        nb = adj[off[s]:off[s + 1]]
        assert np.all(np.diff(nb.astype(np.int64)) > 0), "ascending, unique"
        assert s not in nb
        pairs.update((s, int(w)) for w in nb)
    assert all((w, s) in pairs for s, w in pairs), "symmetric"


def test_random_sites_walk_equals_kdtree():
    """REF/SPEC.md:479 example: both strategies on 1000 random sites, 10^4 queries -> identical."""
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1, 1, (1000, 3))
    off, adj = P.delaunay_adjacency(pts)
    _check_adjacency(off, adj, len(pts))
    assert 8 < off[-1] / len(pts) < 24          # ~15.5 Delaunay neighbours per site in 3-D
    qs = rng.uniform(-1.3, 1.3, (10_000, 3))
    walk, steps = O.batch_walk(pts, off, adj, qs, threads=1)
    kd = O.KdTree(pts)
    want = np.array([kd.nearest(q)[0] for q in qs])
    assert np.array_equal(walk, want)
    brute = np.array([O.nearest_site_brute(pts, q)[0] for q in qs[:500]])
    assert np.array_equal(walk[:500], brute)
    assert steps > 0
    # correctness does not depend on the start (REF/SPEC.md:516)
    for start in (0, 17, 999):
        for q in qs[:200]:
            assert O.walk_nearest(pts, off, adj, q, start)[0] == kd.nearest(q)[0]


def test_walk_ties_lowest_id():
    """REF/SPEC.md:481: equidistant tie (two mirrored sites, query on the bisector) -> lower id; and
    a tie set that is not connected through improving moves (cospherical ring)."""
    pts = np.array([[1.0, 0, 0], [-1.0, 0, 0], [0, 5, 0], [0, -5, 0], [0, 0, 5], [0, 0, -5]])
    off, adj = P.delaunay_adjacency(pts)
    for start in range(len(pts)):
        assert O.walk_nearest(pts, off, adj, [0.0, 0.3, 0.1], start)[0] == 0
    # four sites on a circle around the z axis, ids not in ring order; q on the axis ties all four
    ring = np.array([[1.0, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0]])
    order = [3, 0, 2, 1]
    pts = np.vstack([ring[order], [[0, 0, 9.0], [0, 0, -9.0]]])
    off, adj = P.delaunay_adjacency(pts)
    for start in range(4):
        assert O.walk_nearest(pts, off, adj, [0.0, 0.0, 0.25], start)[0] == 0
    assert O.walk_nearest(pts, off, adj, pts[2], 5)[0] == 2   # q = a site -> that site (REF/SPEC.md:487)


def test_engine_adjacency_and_walk(ico3):
    V, F, h = ico3
    a = h.arrays()
    S = len(a["site_xyz"])
    _check_adjacency(a["adj_offsets"], a["adj_sites"], S)
    rng = np.random.default_rng(3)
    lo, hi = a["domain"][:3], a["domain"][3:]
    # inside the mesh box, anywhere in D, at the sites, and far outside D (walks among sentinels)
    qs = np.concatenate([rng.uniform(-1.3, 1.3, (4000, 3)), rng.uniform(lo, hi, (1000, 3)),
                         V[:200], rng.uniform(-40, 40, (2000, 3)), rng.uniform(-400, 400, (500, 3))])
    walk, _ = O.batch_walk(a["site_xyz"], a["adj_offsets"], a["adj_sites"], qs)
    kd = O.KdTree(a["site_xyz"])
    want = np.array([kd.nearest(q)[0] for q in qs])
    assert np.array_equal(walk, want)


def test_cospherical_icosphere_walk(c1):
    """c1 is exactly cospherical: many near-degenerate Voronoi vertices."""
    V, F, h = c1
    a = h.arrays()
    qs = np.concatenate([P.gen_queries(1, V, F, 0, 3000), V[:100], np.zeros((1, 3))])
    walk, _ = O.batch_walk(a["site_xyz"], a["adj_offsets"], a["adj_sites"], qs)
    kd = O.KdTree(a["site_xyz"])
    want = np.array([kd.nearest(q)[0] for q in qs])
    assert np.array_equal(walk, want)


@pytest.mark.gpu
@pytest.mark.parametrize("fixture,cfg", [("ico3", None), ("c1", 1), ("c2", 2)])
def test_gpu_strategy_neutrality(request, fixture, cfg):
    V, F, h = request.getfixturevalue(fixture)
    rng = np.random.default_rng(5)
    if cfg:
        q = P.gen_queries(cfg, V, F, 0, 200_000)
    else:
        q = rng.uniform(-1.3, 1.3, (50_000, 3))
    a = h.arrays()
    q = np.concatenate([q, V[:300], rng.uniform(a["domain"][:3], a["domain"][3:], (2000, 3)),
                        rng.uniform(-40, 40, (500, 3))])
    eng = P.Engine(h)
    res = {}
    for st in ("grid", "kdtree", "walk"):
        eng.set_nns_strategy(st)
        res[st] = eng.batch_query(q)
    for st in ("kdtree", "walk"):
        for k in ("distance", "closest", "face", "site", "flags"):
            assert getattr(res[st], k).tobytes() == getattr(res["grid"], k).tobytes(), (st, k)
    ref = oracle_checker(a).batch_query(q)
    assert np.array_equal(res["walk"].site, ref["site"])
    assert res["walk"].distance.tobytes() == ref["distance"].tobytes()


@pytest.mark.gpu
def test_gpu_walk_requires_adjacency(ico3):
    """An engine created without desc.adj_offsets refuses the walk strategy (P2M_ERR_INVALID)."""
    import ctypes as C
    from paper_2605_00429_b200 import _lib as L
    V, F, h = ico3
    d = h.desc()
    d.adj_offsets = None
    d.adj_sites = None
    eh = C.c_void_p()
    L.check(L.cuda().p2m_engine_create(C.byref(d), 1, None, C.byref(eh)))
    try:
        assert L.cuda().p2m_set_nns_strategy(eh, 2) == -1
        assert L.cuda().p2m_set_nns_strategy(eh, 1) == 0
        assert L.cuda().p2m_set_nns_strategy(eh, 7) == -1
    finally:
        L.cuda().p2m_engine_destroy(eh)
