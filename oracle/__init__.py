"""CPU oracle for the point-to-mesh query path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It wraps:
  liboracle.so        -- the plain-C restatement (oracle/p2m_oracle.c, cites REF file:line)
  _ref/libp2m_ref.so  -- the reference's own REF/proj/src/geom.cpp (compiled where it lies, never
                         copied) + the same query loop calling p2mx::closest_on_triangle_sq
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
dp = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)

PRUNE_OFF, PRUNE_SAFE, PRUNE_SPEC = 0, 1, 2


class Counters(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("n_queries", "candidates_visited", "exact_evaluations",
                                          "pruned", "fallbacks", "kd_nodes_visited")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


def _p(a, t=dp):
    return a.ctypes.data_as(t)


def _bind(L):
    L.orc_closest_on_triangle_sq.argtypes = [dp] * 6
    L.orc_triangle_bounding_sphere.argtypes = [dp, dp]
    L.orc_kdtree_build.restype = C.c_void_p
    L.orc_kdtree_build.argtypes = [dp, C.c_uint64]
    L.orc_kdtree_free.argtypes = [C.c_void_p]
    L.orc_kdtree_layout.argtypes = [C.c_void_p, u32p, u8p]
    L.orc_nearest_site.restype = C.c_uint32
    L.orc_nearest_site.argtypes = [C.c_void_p, dp, dp, u64p]
    L.orc_nearest_site_brute.restype = C.c_uint32
    L.orc_nearest_site_brute.argtypes = [dp, C.c_uint64, dp, dp]
    L.orc_brute_force_closest.restype = C.c_uint32
    L.orc_brute_force_closest.argtypes = [dp, C.c_uint64, dp, dp, dp]
    L.orc_batch_brute_force.argtypes = [dp, C.c_uint64, dp, C.c_uint64, C.c_int, dp, dp, u32p]
    L.orc_ctx_create.restype = C.c_void_p
    L.orc_ctx_create.argtypes = [C.c_uint64, dp, u8p, C.c_uint64, dp, dp, u64p, u32p, dp]
    L.orc_ctx_free.argtypes = [C.c_void_p]
    L.orc_batch_query.argtypes = [C.c_void_p, dp, C.c_uint64, C.c_int, C.c_int, dp, dp, u32p, u32p, u32p,
                                  u64p, C.POINTER(Counters)]
    L.orc_walk_nearest.restype = C.c_uint32
    L.orc_walk_nearest.argtypes = [dp, u64p, u32p, C.c_uint64, dp, C.c_uint32, dp, u64p]
    L.orc_batch_walk.argtypes = [dp, u64p, u32p, C.c_uint64, dp, C.c_uint64, C.c_int, u32p, u64p]
    L.orc_max_threads.restype = C.c_int
    L.orc_uses_reference_kernel.restype = C.c_int
    return L


_libs = {}


def lib(reference: bool = False):
    """reference=False: the restatement; True: the reference-compiled build (oracle/_ref)."""
    key = bool(reference)
    if key not in _libs:
        path = os.path.join(HERE, "_ref", "libp2m_ref.so") if reference else os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run `make -C oracle` (the _ref build needs /root/reference)")
        L = _bind(C.CDLL(path))
        if reference:
            L.p2mref_closest_on_triangle_sq.argtypes = [dp] * 6
            L.p2mref_triangle_bounding_sphere.argtypes = [dp, dp]
            L.p2mref_triangle_bounding_sphere.restype = C.c_int
            L.p2mref_point_triangle_distance.argtypes = [dp, dp, dp, dp]
            L.p2mref_point_triangle_distance.restype = C.c_int
            L.p2mref_sphere_triangle_intersect.argtypes = [dp, dp]
            L.p2mref_sphere_triangle_intersect.restype = C.c_int
            L.p2mref_tetra_circumcenter.argtypes = [dp] * 5
            L.p2mref_tetra_circumcenter.restype = C.c_int
            L.p2mref_orient3d.argtypes = [dp] * 4
            L.p2mref_orient3d.restype = C.c_int
            L.p2mref_in_sphere.argtypes = [dp] * 5
            L.p2mref_in_sphere.restype = C.c_int
            L.p2mref_aabb_scaled.argtypes = [dp, dp, C.c_double, C.c_double, dp]
        _libs[key] = L
    return _libs[key]


def have_reference() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libp2m_ref.so"))


def closest_on_triangle_sq(q, a, b, c, reference=False):
    L = lib(reference)
    q, a, b, c = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, a, b, c))
    d2 = np.zeros(1); p = np.zeros(3)
    fn = L.p2mref_closest_on_triangle_sq if reference else L.orc_closest_on_triangle_sq
    fn(_p(q), _p(a), _p(b), _p(c), _p(d2), _p(p))
    return float(d2[0]), p


def triangle_bounding_sphere(tri, reference=False):
    L = lib(reference)
    t = np.ascontiguousarray(tri, dtype=np.float64).reshape(9)
    out = np.zeros(4)
    if reference:
        rc = L.p2mref_triangle_bounding_sphere(_p(t), _p(out))
        if rc != 0:
            raise ValueError("GeometryError: degenerate triangle")
    else:
        L.orc_triangle_bounding_sphere(_p(t), _p(out))
    return out


def brute_force_closest(tri, q, reference=False):
    """(d2, point, face) -- linear scan, lowest face id on ties (REF/SPEC.md:536-544)."""
    L = lib(reference)
    tri = np.ascontiguousarray(tri, dtype=np.float64).reshape(-1, 9)
    q = np.ascontiguousarray(q, dtype=np.float64)
    d2 = np.zeros(1); p = np.zeros(3)
    f = L.orc_brute_force_closest(_p(tri), len(tri), _p(q), _p(d2), _p(p))
    return float(d2[0]), p, int(f)


def batch_brute_force(tri, q, reference=False, threads=0):
    """brute_force_closest for every row of q (OpenMP): {'d2', 'closest', 'face'}."""
    L = lib(reference)
    tri = np.ascontiguousarray(tri, dtype=np.float64).reshape(-1, 9)
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
    n = len(q)
    d2 = np.zeros(n); p = np.zeros((n, 3)); f = np.zeros(n, np.uint32)
    L.orc_batch_brute_force(_p(tri), len(tri), _p(q), n, threads, _p(d2), _p(p), _p(f, u32p))
    return {"d2": d2, "closest": p, "face": f}


def nearest_site_brute(sites, q, reference=False):
    L = lib(reference)
    s = np.ascontiguousarray(sites, dtype=np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(q, dtype=np.float64)
    d2 = np.zeros(1)
    return int(L.orc_nearest_site_brute(_p(s), len(s), _p(q), _p(d2))), float(d2[0])


class KdTree:
    def __init__(self, sites, reference=False):
        self._L = lib(reference)
        self.sites = np.ascontiguousarray(sites, dtype=np.float64).reshape(-1, 3)
        self._t = self._L.orc_kdtree_build(_p(self.sites), len(self.sites))

    def __del__(self):
        if getattr(self, "_t", None):
            self._L.orc_kdtree_free(self._t)
            self._t = None

    def layout(self):
        n = len(self.sites)
        ns = np.zeros(n, np.uint32); nd = np.zeros(n, np.uint8)
        self._L.orc_kdtree_layout(self._t, _p(ns, u32p), _p(nd, u8p))
        return ns, nd

    def nearest(self, q):
        q = np.ascontiguousarray(q, dtype=np.float64)
        d2 = np.zeros(1); vis = np.zeros(1, np.uint64)
        s = self._L.orc_nearest_site(self._t, _p(q), _p(d2), _p(vis, u64p))
        return int(s), float(d2[0]), int(vis[0])


class OracleEngine:
    """query_distance / batch_query (REF/SPEC.md:488-505) on the same engine arrays the GPU gets."""

    def __init__(self, arrays: dict, reference=False):
        self._L = lib(reference)
        a = arrays
        self._keep = {
            "site_xyz": np.ascontiguousarray(a["site_xyz"], dtype=np.float64),
            "site_kind": np.ascontiguousarray(a["site_kind"], dtype=np.uint8),
            "tri": np.ascontiguousarray(a["tri"], dtype=np.float64),
            "sphere": np.ascontiguousarray(a["sphere"], dtype=np.float64),
            "off": np.ascontiguousarray(a["list_offsets"], dtype=np.uint64),
            "faces": np.ascontiguousarray(a["list_faces"], dtype=np.uint32),
            "domain": np.ascontiguousarray(a["domain"], dtype=np.float64),
        }
        k = self._keep
        if len(k["faces"]) == 0:
            k["faces"] = np.zeros(1, np.uint32)
        self.n_sites = len(k["site_kind"])
        self.n_faces = len(k["sphere"])
        self._c = self._L.orc_ctx_create(self.n_sites, _p(k["site_xyz"]), _p(k["site_kind"], u8p), self.n_faces,
                                         _p(k["tri"]), _p(k["sphere"]), _p(k["off"], u64p), _p(k["faces"], u32p),
                                         _p(k["domain"]))
        if not self._c:
            raise MemoryError("orc_ctx_create failed")

    def __del__(self):
        if getattr(self, "_c", None):
            self._L.orc_ctx_free(self._c)
            self._c = None

    def batch_query(self, q, prune=PRUNE_SAFE, threads=0, per_query=False):
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
        n = len(q)
        dist = np.empty(n); cp = np.empty((n, 3)); face = np.empty(n, np.uint32)
        site = np.empty(n, np.uint32); flags = np.empty(n, np.uint32)
        pq = np.empty((n, 3), np.uint64) if per_query else None
        cnt = Counters()
        self._L.orc_batch_query(self._c, _p(q), n, prune, threads, _p(dist), _p(cp), _p(face, u32p),
                                _p(site, u32p), _p(flags, u32p), _p(pq, u64p) if per_query else None,
                                C.byref(cnt))
        out = {"distance": dist, "closest": cp, "face": face, "site": site, "flags": flags,
               "counters": cnt.as_dict()}
        if per_query:
            out["per_query"] = pq
        return out


def walk_nearest(sites, adj_off, adj, q, start=0):
    """DelaunayWalk nearest site (REF/SPEC.md:476): (site, d2, steps)."""
    xyz = np.ascontiguousarray(sites, dtype=np.float64).reshape(-1, 3)
    ao = np.ascontiguousarray(adj_off, dtype=np.uint64)
    aj = np.ascontiguousarray(adj, dtype=np.uint32)
    qq = np.ascontiguousarray(q, dtype=np.float64).reshape(3)
    d2 = C.c_double()
    st = C.c_uint64(0)
    s = lib().orc_walk_nearest(_p(xyz), _p(ao, u64p), _p(aj, u32p), len(xyz), _p(qq), int(start),
                               C.byref(d2), C.byref(st))
    return int(s), d2.value, int(st.value)


def batch_walk(sites, adj_off, adj, q, threads=0):
    """Batch DelaunayWalk with the SPEC's per-thread warm start (REF/SPEC.md:516): (sites, steps)."""
    xyz = np.ascontiguousarray(sites, dtype=np.float64).reshape(-1, 3)
    ao = np.ascontiguousarray(adj_off, dtype=np.uint64)
    aj = np.ascontiguousarray(adj, dtype=np.uint32)
    qq = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
    out = np.empty(len(qq), np.uint32)
    st = C.c_uint64(0)
    lib().orc_batch_walk(_p(xyz), _p(ao, u64p), _p(aj, u32p), len(xyz), _p(qq), len(qq), threads,
                         _p(out, u32p), C.byref(st))
    return out, int(st.value)


def max_threads(reference=False) -> int:
    return int(lib(reference).orc_max_threads())
