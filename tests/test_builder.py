"""Host build phase (REF/SPEC.md:112-456): the structure the query path consumes.

The load-bearing property is the superset invariant (REF/SPEC.md:435): for a query q in D with
nearest site v, the brute-force closest face (REF/SPEC.md:536-544) is in table(v).  Everything the
GPU computes is checked against the oracle on these tables; this file checks the tables themselves.
"""
import ctypes as C
import os
import tempfile

import numpy as np
import pytest

import oracle as O
import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L

needs_ref = pytest.mark.skipif(not O.have_reference(), reason="oracle/_ref not built")

TET_V = np.array([[1.0, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]])
TET_F = np.array([[0, 1, 2], [0, 3, 1], [0, 2, 3], [1, 3, 2]], np.uint32)
TRI_V = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
TRI_F = np.array([[0, 1, 2]], np.uint32)


def bumpy_sphere(level=3, seed=0, amp=0.05):
    V, F = P.icosphere(level)
    rng = np.random.default_rng(seed)
    return V * (1.0 + amp * rng.standard_normal((len(V), 1))), F


def superset_check(h, nq=1500, seed=0, box=None):
    a = h.arrays()
    tri = a["tri"].reshape(-1, 9)
    sites = a["site_xyz"]
    rng = np.random.default_rng(seed)
    lo, hi = (a["domain"][:3], a["domain"][3:]) if box is None else box
    qs = rng.uniform(lo, hi, size=(nq, 3))
    kd = O.KdTree(sites)
    off, lf = a["list_offsets"], a["list_faces"]
    bad = 0
    for q in qs:
        s, _, _ = kd.nearest(q)
        assert a["site_kind"][s] != L.SITE_SENTINEL, "a sentinel is nearest inside D"
        d2, _, f = O.brute_force_closest(tri, q)
        lst = lf[off[s]:off[s + 1]]
        if f not in lst:
            # a tie with another listed face at exactly the same distance is fine
            ok = any(O.closest_on_triangle_sq(q, *a["tri"][g])[0] == d2 for g in lst)
            bad += not ok
    return bad


@pytest.mark.parametrize("mesh", ["tri", "tet", "ico2", "bumpy3"])
def test_superset_property(mesh):
    V, F = {"tri": (TRI_V, TRI_F), "tet": (TET_V, TET_F), "ico2": P.icosphere(2), "bumpy3": bumpy_sphere()}[mesh]
    h = P.HostEngine.build(V, F)
    assert superset_check(h) == 0
    aabb = (V.min(0) - 0.3 * np.ptp(V, 0), V.max(0) + 0.3 * np.ptp(V, 0))
    assert superset_check(h, seed=1, box=aabb) == 0


def test_superset_property_c1(c1):
    V, F, h = c1
    q_box = (V.min(0) * 1.2, V.max(0) * 1.2)
    assert superset_check(h, nq=400, seed=3, box=q_box) == 0


def test_tables_sorted_unique_and_incident(ico3):
    V, F, h = ico3
    a = h.arrays()
    off, lf, kind = a["list_offsets"], a["list_faces"], a["site_kind"]
    nv = len(V)
    inc = [[] for _ in range(nv)]
    for f, t in enumerate(F):
        for v in t:
            inc[v].append(f)
    for s in range(len(kind)):
        lst = lf[off[s]:off[s + 1]]
        if kind[s] == L.SITE_SENTINEL:
            assert len(lst) == 0  # REF/SPEC.md:418
            continue
        assert len(lst) > 0  # REF/SPEC.md:393
        assert np.all(np.diff(lst.astype(np.int64)) > 0)  # sorted, deduplicated (REF/SPEC.md:392)
        if kind[s] == L.SITE_MESH_VERTEX:
            assert set(inc[s]) <= set(lst.tolist())  # REF/SPEC.md:421


def test_site_order_and_sentinels(ico3):
    V, F, h = ico3
    a = h.arrays()
    kind = a["site_kind"]
    nv = len(V)
    assert np.all(kind[:nv] == L.SITE_MESH_VERTEX) and np.array_equal(a["site_xyz"][:nv], V)
    assert np.all(kind[nv:nv + 8] == L.SITE_SENTINEL) and np.all(kind[nv + 8:] == L.SITE_AUXILIARY)
    D = a["domain"]
    c, h4 = (D[:3] + D[3:]) / 2, (D[3:] - D[:3]) * 2.0  # sentinels at corners of D scaled 4x
    assert np.allclose(np.abs(a["site_xyz"][nv:nv + 8] - c), h4)
    refs = a["site_refs"]
    assert np.all(np.isnan(refs[:nv + 8]))
    # every auxiliary reference lies on the mesh (REF/SPEC.md:363)
    tri = a["tri"].reshape(-1, 9)
    for s in range(nv + 8, len(kind), max(1, (len(kind) - nv - 8) // 25)):
        d2, _, _ = O.brute_force_closest(tri, refs[s])
        assert d2 <= (1e-10 * np.linalg.norm(D[3:] - D[:3])) ** 2


@needs_ref
def test_face_spheres_bit_identical_to_reference(c2):
    V, F, h = c2
    a = h.arrays()
    for f in range(0, len(F), 97):
        ref = O.triangle_bounding_sphere(a["tri"][f], reference=True)
        assert ref.tobytes() == a["sphere"][f].tobytes()


def test_face_spheres_contain_triangles(c2):
    V, F, h = c2
    a = h.arrays()
    d = np.linalg.norm(a["tri"] - a["sphere"][:, None, :3], axis=2)
    assert np.all(d <= a["sphere"][:, 3:4] * (1 + 1e-12))  # REF/SPEC.md:91


def test_augmentation_behaviour():
    # icosphere: dense central Voronoi-vertex cluster -> auxiliary sites inserted (REF/SPEC.md:357)
    V, F = P.icosphere(4)
    h = P.HostEngine.build(V, F)
    st = h.stats()
    assert st["n_aux_sites"] >= 15 and 1 <= st["rounds_used"] <= 3
    a = h.arrays()
    aux = a["site_xyz"][a["site_kind"] == L.SITE_AUXILIARY]
    assert np.min(np.linalg.norm(aux, axis=1)) < st["tau"]  # one cluster sits at the centre
    # augmentation off vs on: the tables shrink dramatically (REF/Table 4 direction)
    h0 = P.HostEngine.build(V, F, P.BuildConfig(augment=False))
    assert h0.stats()["n_aux_sites"] == 0
    assert h0.stats()["list_avg"] > 5 * st["list_avg"]
    # k = 1 saturates at max_rounds without error (REF/SPEC.md:358)
    hk = P.HostEngine.build(*P.icosphere(2), P.BuildConfig(k=1, max_rounds=2))
    assert hk.stats()["rounds_used"] <= 2


def test_aux_corner_union_is_subset_and_valid():
    V, F = bumpy_sphere(3, seed=2)
    h1 = P.HostEngine.build(V, F, P.BuildConfig(aux_corner_union=False))
    h2 = P.HostEngine.build(V, F, P.BuildConfig(aux_corner_union=True))
    assert superset_check(h1, nq=800) == 0
    a1, a2 = h1.arrays(), h2.arrays()
    assert np.array_equal(a1["site_xyz"], a2["site_xyz"])
    for s in np.flatnonzero(a1["site_kind"] == L.SITE_AUXILIARY):
        l1 = set(a1["list_faces"][a1["list_offsets"][s]:a1["list_offsets"][s + 1]].tolist())
        l2 = set(a2["list_faces"][a2["list_offsets"][s]:a2["list_offsets"][s + 1]].tolist())
        assert l2 <= l1  # REF/SPEC.md:413
    assert superset_check(h2, nq=800) == 0


def test_build_is_deterministic(ico3):
    V, F, h = ico3
    h2 = P.HostEngine.build(V, F)
    a, b = h.arrays(), h2.arrays()
    for k in ("site_xyz", "site_kind", "list_offsets", "list_faces", "sphere", "tri", "domain"):
        assert a[k].tobytes() == b[k].tobytes(), k  # REF/SPEC.md:438, 605


def test_validate_mesh():
    # duplicate vertex merged, faces reindexed (REF/SPEC.md:138)
    V = np.vstack([TET_V, TET_V[:1]])
    F = TET_F.copy()
    F[0, 0] = 4
    h = P.HostEngine.build(V, F)
    st = h.stats()
    assert st["merged_vertices"] == 1 and st["n_vertices"] == 4
    v2, f2 = h.mesh()
    assert np.array_equal(v2, TET_V) and np.array_equal(f2, TET_F)
    # one zero-area face among the faces is removed and reported (REF/SPEC.md:139)
    V3 = np.vstack([TET_V, [[0.0, 0, 0], [1.0, 0, 0], [2.0, 0, 0]]])
    F3 = np.vstack([TET_F, [[4, 5, 6]]]).astype(np.uint32)
    h3 = P.HostEngine.build(V3, F3)
    assert h3.stats()["removed_faces"] == 1 and h3.stats()["n_faces"] == 4
    with pytest.raises(P.P2MError):
        P.HostEngine.build(V3, F3, P.BuildConfig(strict_mesh=True))
    # clean mesh unchanged (REF/SPEC.md:140); all faces degenerate -> error
    assert P.HostEngine.build(TET_V, TET_F).stats()["removed_faces"] == 0
    with pytest.raises(P.P2MError):
        P.HostEngine.build(np.zeros((3, 3)), np.array([[0, 1, 2]], np.uint32))
    with pytest.raises(P.P2MError):
        P.HostEngine.build(TET_V, np.array([[0, 1, 9]], np.uint32))


def test_single_triangle_tables():
    h = P.HostEngine.build(TRI_V, TRI_F)
    a = h.arrays()
    for s in np.flatnonzero(a["site_kind"] != L.SITE_SENTINEL):
        assert a["list_faces"][a["list_offsets"][s]:a["list_offsets"][s + 1]].tolist() == [0]  # REF/SPEC.md:403


def test_cell_corners_equidistance():
    V, F = bumpy_sphere(2, seed=4)
    h = P.HostEngine.build(V, F)
    a = h.arrays()
    sites = a["site_xyz"]
    for s in range(0, len(V), 13):
        u = h.cell_corners(s)
        assert len(u) >= 4
        dv = np.linalg.norm(u - sites[s], axis=1)
        dmin = np.min(np.linalg.norm(u[:, None, :] - sites[None, :, :], axis=2), axis=1)
        assert np.all(dv <= dmin + 1e-9 * (1 + dv))  # REF/SPEC.md:272, 286


def test_save_load_round_trip(ico3):
    V, F, h = ico3
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "e.p2mx")
        h.save(path)
        with open(path, "rb") as f:
            assert f.read(4) == b"P2MX"
        h2 = P.HostEngine.load(path, V, F)
        a, b = h.arrays(), h2.arrays()
        for k in ("site_xyz", "site_kind", "list_offsets", "list_faces", "sphere", "tri", "domain",
                  "adj_offsets", "adj_sites"):
            assert a[k].tobytes() == b[k].tobytes(), k
        q = np.random.default_rng(0).uniform(-1.2, 1.2, size=(500, 3))
        r1 = O.OracleEngine(a).batch_query(q)
        r2 = O.OracleEngine(b).batch_query(q)
        assert r1["distance"].tobytes() == r2["distance"].tobytes()  # REF/SPEC.md:590, 641
        V2 = V.copy()
        V2[0, 0] += 1e-3
        with pytest.raises(P.P2MError, match="hash"):
            P.HostEngine.load(path, V2, F)  # wrong mesh hash
        with open(path, "rb") as f:
            blob = f.read()
        with open(path, "wb") as f:
            f.write(blob[: len(blob) // 2])
        with pytest.raises(P.P2MError):
            P.HostEngine.load(path, V, F)  # truncated


def test_load_rejects_corrupt_contents(ico3, tmp_path):
    """EngineIndexFile v4: config/stats are stored field by field, and load checks every
    id and offset against its range -- a face id >= F, a bad site kind or non-monotone offsets fail
    with P2M_ERR_IO instead of reaching the table or query paths."""
    V, F, h = ico3
    path = str(tmp_path / "e.p2mx")
    h.save(path)
    blob = bytearray(open(path, "rb").read())
    a = h.arrays()
    S = len(a["site_kind"])
    head = 4 + 4 + 8 + 48 + (6 * 4 + 3 * 8) + (8 * 8 + 4 + 2 * 8 + 2 * 8 + 8 + 4 * 8 + 8) + 8
    kind_at = head
    off_at = head + S + 48 * S + 32
    lists_at = off_at + 8 * (S + 1)
    assert bytes(blob[kind_at:kind_at + S]) == a["site_kind"].tobytes()
    assert bytes(blob[lists_at:lists_at + 8]) == a["list_faces"][:2].tobytes()
    for name, at, val in (("face ids", lists_at, b"\xff\xff\xff\xff"), ("site kinds", kind_at + 3, b"\x07"),
                          ("table offsets", off_at + 8 * 5, b"\x00" * 8)):
        bad = bytearray(blob)
        bad[at:at + len(val)] = val
        p2 = str(tmp_path / "bad.p2mx")
        open(p2, "wb").write(bytes(bad))
        with pytest.raises(P.P2MError, match="corrupt") as ei:
            P.HostEngine.load(p2, V, F)
        assert ei.value.code == -6 and name.split()[0] in str(ei.value), name


def test_config_meshes_and_queries():
    V, F = P.mesh_config(1)
    assert (len(V), len(F)) == (10242, 20480)
    V3, F3 = P.mesh_config(3)
    assert (len(V3), len(F3)) == (132100, 264192)
    q = P.gen_queries(1, V, F, 0, 2000)
    q2 = P.gen_queries(1, V, F, 1000, 1000)
    assert np.array_equal(q[1000:], q2)  # counter-based: slices are consistent
    lo, hi = V.min(0), V.max(0)
    c, hh = (lo + hi) / 2, (hi - lo) * 0.6
    assert np.all(np.abs(q - c) <= hh + 1e-12)
    V2, F2 = P.mesh_config(2)
    q = P.gen_queries(2, V2, F2, 0, 4000)
    r = np.linalg.norm(q[1::2], axis=1)
    assert np.abs(r - 1).mean() < 0.05  # odd rows are near-surface samples


@pytest.mark.slow
def test_config_meshes_large():
    V4, F4 = P.mesh_config(4)
    assert (len(V4), len(F4)) == (524288, 1048576)
    V5, F5 = P.mesh_config(5)
    assert (len(V5), len(F5)) == (655362, 1310720)
    assert np.min(np.linalg.norm(V5, axis=1)) > 0.05
