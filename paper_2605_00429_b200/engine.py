"""Host-side mirror of the reference's build-then-query API for the point-to-mesh query path.

Reference interface (REF = /root/reference, spec-only for everything but geometry):
  build      -> cmd_build pipeline                 REF/SPEC.md:598-606   -> HostEngine.build
  query      -> build_nns_index                    REF/SPEC.md:473-481   -> Engine(...)
             -> nearest_site                       REF/SPEC.md:482-487   -> Engine.nearest_site
             -> query_distance                     REF/SPEC.md:488-496   -> Engine.query_distance
             -> batch_query                        REF/SPEC.md:497-505   -> Engine.batch_query
  errors     -> "engine not built" (REF/SPEC.md:492) -> P2MError(P2M_ERR_NOT_BUILT); out-of-domain
                queries are never errors (REF/SPEC.md:611), they are flagged per row.

The query itself always runs on the GPU through libp2m_cuda.so; there is no CPU path here.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

__all__ = [
    "BuildConfig",
    "HostEngine",
    "Engine",
    "QueryResult",
    "BatchResult",
    "mesh_config",
    "icosphere",
    "gen_queries",
    "gen_uniform",
]


@dataclasses.dataclass
class BuildConfig:
    """AugmentationConfig + cli flags (REF/SPEC.md:313-316, 367, 656)."""

    augment: bool = True
    alpha: float = 4.0
    k: int = 24
    rho: float = 0.75
    max_rounds: int = 3
    domain_scale: float = 10.0
    n_threads: int = 0
    strict_mesh: bool = False
    aux_corner_union: bool = True

    def to_c(self) -> L.BuildConfig:
        c = L.BuildConfig()
        L.host().p2m_build_config_default(C.byref(c))
        c.augment = int(self.augment)
        c.alpha = self.alpha
        c.k = self.k
        c.rho = self.rho
        c.max_rounds = self.max_rounds
        c.domain_scale = self.domain_scale
        c.n_threads = self.n_threads
        c.strict_mesh = int(self.strict_mesh)
        c.aux_corner_union = int(self.aux_corner_union)
        return c


def _as_mesh(vertices, faces):
    v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
    f = np.ascontiguousarray(faces, dtype=np.uint32).reshape(-1, 3)
    return v, f


class HostEngine:
    """The preprocessed structure: validated mesh, sites, interception tables, face spheres."""

    def __init__(self, handle: C.c_void_p, keep=()):
        self._h = handle
        self._keep = keep

    @classmethod
    def build(cls, vertices, faces, config: Optional[BuildConfig] = None,
              table_device: Optional[int] = None) -> "HostEngine":
        """cmd_build (REF/SPEC.md:598-606).  table_device=k runs build_all_tables on GPU k
        (p2m_build_device, bit-identical tables); None keeps the whole build on host threads."""
        v, f = _as_mesh(vertices, faces)
        cfg = (config or BuildConfig()).to_c()
        h = C.c_void_p()
        if table_device is None:
            L.check(L.host().p2m_build(L.ptr(v), len(v), L.ptr(f, L.u32p), len(f), C.byref(cfg), C.byref(h)))
        else:
            L.check(L.cuda().p2m_build_device(L.ptr(v), len(v), L.ptr(f, L.u32p), len(f), C.byref(cfg),
                                              int(table_device), C.byref(h)))
        return cls(h)

    @classmethod
    def build_with(cls, vertices, faces, table_fn, config: Optional[BuildConfig] = None) -> "HostEngine":
        """p2m_build_with: table_fn(job) -> (off[S+1] uint64, lists uint32) runs the table job
        (include/p2m.h p2m_table_job, exposed as numpy arrays)."""
        v, f = _as_mesh(vertices, faces)
        cfg = (config or BuildConfig()).to_c()
        h = C.c_void_p()
        libc = C.CDLL(None)
        libc.malloc.restype = C.c_void_p
        libc.malloc.argtypes = [C.c_size_t]
        err = []

        def _cb(ctx, job_p, off_p, lists_pp):
            try:
                j = C.cast(job_p, C.POINTER(L.TableJob)).contents
                S, NF, NN = j.n_sites, j.n_faces, j.n_nodes
                boff = np.ctypeslib.as_array(j.ball_off, (S + 1,)).copy()
                nb = int(boff[-1])
                job = {
                    "ball_off": boff,
                    "balls": np.ctypeslib.as_array(j.balls, (max(nb, 1) * 4,))[: 4 * nb].reshape(-1, 4).copy(),
                    "tri": np.ctypeslib.as_array(j.tri, (max(NF, 1) * 9,))[: 9 * NF].reshape(-1, 9).copy(),
                    "node_box": np.ctypeslib.as_array(j.node_box, (max(NN, 1) * 6,))[: 6 * NN].reshape(-1, 6).copy(),
                    "node_meta": np.ctypeslib.as_array(j.node_meta, (max(NN, 1) * 3,))[: 3 * NN].reshape(-1, 3).copy(),
                    "perm": np.ctypeslib.as_array(j.perm, (max(NF, 1),))[:NF].copy(),
                }
                off, lists = table_fn(job)
                off = np.ascontiguousarray(off, dtype=np.uint64)
                lists = np.ascontiguousarray(lists, dtype=np.uint32)
                C.memmove(off_p, off.ctypes.data, 8 * (S + 1))
                buf = libc.malloc(max(4 * len(lists), 4))
                if len(lists):
                    C.memmove(buf, lists.ctypes.data, 4 * len(lists))
                lists_pp[0] = C.cast(buf, L.u32p)
                return 0
            except Exception as e:  # surfaced through p2m_last_error
                err.append(e)
                return -7

        cb = L.TABLE_FN(_cb)
        rc = L.host().p2m_build_with(L.ptr(v), len(v), L.ptr(f, L.u32p), len(f), C.byref(cfg),
                                      C.cast(cb, C.c_void_p), None, C.byref(h))
        if err:
            raise err[0]
        L.check(rc)
        return cls(h)

    @classmethod
    def load(cls, path: str, vertices, faces) -> "HostEngine":
        v, f = _as_mesh(vertices, faces)
        h = C.c_void_p()
        L.check(L.host().p2m_host_engine_load(path.encode(), L.ptr(v), len(v), L.ptr(f, L.u32p), len(f), C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        L.check(L.host().p2m_host_engine_save(self._h, path.encode()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                L.host().p2m_host_engine_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def desc(self) -> L.EngineDesc:
        d = L.EngineDesc()
        L.check(L.host().p2m_host_engine_desc(self._h, C.byref(d)))
        return d

    def stats(self) -> dict:
        s = L.BuildStats()
        L.check(L.host().p2m_host_engine_stats(self._h, C.byref(s)))
        return s.as_dict()

    def arrays(self) -> dict:
        """Zero-copy numpy views of the engine arrays (valid while this object lives)."""
        d = self.desc()
        S, F = int(d.n_sites), int(d.n_faces)
        off = np.ctypeslib.as_array(d.list_offsets, shape=(S + 1,))
        L_ = int(off[-1])
        out = {
            "site_xyz": np.ctypeslib.as_array(d.site_xyz, shape=(S, 3)),
            "site_kind": np.ctypeslib.as_array(d.site_kind, shape=(S,)),
            "tri": np.ctypeslib.as_array(d.tri_xyz, shape=(F, 3, 3)),
            "sphere": np.ctypeslib.as_array(d.face_sphere, shape=(F, 4)),
            "list_offsets": off,
            "list_faces": np.ctypeslib.as_array(d.list_faces, shape=(L_,)) if L_ else np.zeros(0, np.uint32),
            "domain": np.array(list(d.domain_min) + list(d.domain_max)),
        }
        if d.adj_offsets:
            ao = np.ctypeslib.as_array(d.adj_offsets, shape=(S + 1,))
            out["adj_offsets"] = ao
            out["adj_sites"] = (np.ctypeslib.as_array(d.adj_sites, shape=(int(ao[-1]),)) if int(ao[-1])
                                else np.zeros(0, np.uint32))
        refs = L.dp()
        L.check(L.host().p2m_host_engine_site_refs(self._h, C.byref(refs)))
        out["site_refs"] = np.ctypeslib.as_array(refs, shape=(S, 3))
        return out

    def mesh(self):
        v = L.dp(); f = L.u32p(); nv = C.c_uint64(); nf = C.c_uint64()
        L.check(L.host().p2m_host_engine_mesh(self._h, C.byref(v), C.byref(nv), C.byref(f), C.byref(nf)))
        return (np.ctypeslib.as_array(v, shape=(nv.value, 3)).copy(),
                np.ctypeslib.as_array(f, shape=(nf.value, 3)).copy())

    def cell_corners(self, site: int) -> np.ndarray:
        n = C.c_uint64()
        L.check(L.host().p2m_host_engine_cell_corners(self._h, site, None, 0, C.byref(n)))
        out = np.zeros((n.value, 3))
        L.check(L.host().p2m_host_engine_cell_corners(self._h, site, L.ptr(out), n.value, C.byref(n)))
        return out

    def closest_point_bvh(self, q):
        """bvh_closest_point (REF/SPEC.md:201-209), host BVH -- used by tests only."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        d2 = C.c_double(); p = np.zeros(3); f = C.c_uint32()
        L.check(L.host().p2m_host_closest_point(self._h, L.ptr(q), C.byref(d2), L.ptr(p), C.byref(f)))
        return d2.value, p, f.value


@dataclasses.dataclass
class QueryResult:
    """QueryResult (REF/SPEC.md:467-470)."""

    distance: float
    closest: np.ndarray
    face: int
    site: int
    flags: int
    fallback: bool


@dataclasses.dataclass
class BatchResult:
    distance: np.ndarray   # (n,) fp64
    closest: np.ndarray    # (n, 3) fp64
    face: np.ndarray       # (n,) u32
    site: np.ndarray       # (n,) u32
    flags: np.ndarray      # (n,) u32
    counters: dict


class Engine:
    """Device engine: the structure replicated on one or more GPUs (one-time peer copy)."""

    def __init__(self, host_engine: HostEngine, devices: Sequence[int] = (0,)):
        if host_engine is None or not host_engine.handle:
            raise L.P2MError(-3, "engine not built")
        self.host_engine = host_engine
        d = host_engine.desc()
        ids = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        L.check(L.cuda().p2m_engine_create(C.byref(d), len(devices), ids, C.byref(h)))
        self._h = h
        self.devices = tuple(devices)

    @classmethod
    def from_desc(cls, desc: L.EngineDesc, devices: Sequence[int] = (0,), keep=()) -> "Engine":
        """An engine from a caller-filled p2m_engine_desc (the drop-in path of an external builder,
        INTEGRATION.md); `keep` holds the arrays its pointers refer to until creation returns."""
        self = cls.__new__(cls)
        self.host_engine = None
        ids = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        L.check(L.cuda().p2m_engine_create(C.byref(desc), len(devices), ids, C.byref(h)))
        self._h = h
        self.devices = tuple(devices)
        return self

    @classmethod
    def load(cls, path: str, devices: Sequence[int] = (0,)) -> "Engine":
        """An engine straight from a device image file (p2m_engine_load): no host engine, no
        re-packing; bit-identical queries to the engine that was saved."""
        self = cls.__new__(cls)
        self.host_engine = None
        ids = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        L.check(L.cuda().p2m_engine_load(path.encode(), len(devices), ids, C.byref(h)))
        self._h = h
        self.devices = tuple(devices)
        return self

    def save(self, path: str) -> None:
        """Write the packed device layout (p2m_engine_save, "P2MD" v1)."""
        L.check(L.cuda().p2m_engine_save(self.handle, path.encode()))

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                L.cuda().p2m_engine_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    __del__ = close

    @property
    def handle(self):
        if not self._h:
            raise L.P2MError(-3, "engine not built")
        return self._h

    def info(self) -> dict:
        n = C.c_int(); ms = C.c_double(); b = C.c_uint64()
        L.check(L.cuda().p2m_engine_info(self.handle, C.byref(n), C.byref(ms), C.byref(b)))
        return {"n_devices": n.value, "replicate_ms": ms.value, "device_bytes": b.value}

    def batch_query(self, points, counters: bool = True) -> BatchResult:
        """batch_query (REF/SPEC.md:497-505) on host arrays (p2m_query; pageable numpy memory goes
        through the library's pinned bounce rings).  counters=False skips the counters pass."""
        q = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        n = len(q)
        dist = np.empty(n); cp = np.empty((n, 3))
        face = np.empty(n, np.uint32); site = np.empty(n, np.uint32); flags = np.empty(n, np.uint32)
        cnt = L.Counters()
        L.check(L.cuda().p2m_query(self.handle, L.ptr(q), n, L.ptr(dist), L.ptr(cp), L.ptr(face, L.u32p),
                                   L.ptr(site, L.u32p), L.ptr(flags, L.u32p), C.byref(cnt) if counters else None))
        return BatchResult(dist, cp, face, site, flags, cnt.as_dict() if counters else {})

    def query_distance(self, q) -> QueryResult:
        r = self.batch_query(np.asarray(q, dtype=np.float64).reshape(1, 3))
        return QueryResult(float(r.distance[0]), r.closest[0], int(r.face[0]), int(r.site[0]),
                           int(r.flags[0]), bool(r.flags[0] & L.FLAG_FALLBACK))

    def nearest_site(self, points) -> np.ndarray:
        return self.batch_query(points).site

    NNS = {"grid": 0, "kdtree": 1, "walk": 2}

    def set_nns_strategy(self, strategy: str) -> None:
        """NearestSiteIndex strategy (REF/SPEC.md:473-481): 'grid' (default), 'kdtree' or 'walk'
        (DelaunayWalk).  Results never depend on it (strategy neutrality, REF/SPEC.md:510)."""
        L.check(L.cuda().p2m_set_nns_strategy(self.handle, self.NNS[strategy]))


# ---- synthetic workloads -------------------------------------------------------------------

def _take_mesh(v: L.dp, nv, f: L.u32p, nf):
    V = np.ctypeslib.as_array(v, shape=(nv.value, 3)).copy()
    F = np.ctypeslib.as_array(f, shape=(nf.value, 3)).copy()
    L.host().p2m_free(C.cast(v, C.c_void_p))
    L.host().p2m_free(C.cast(f, C.c_void_p))
    return V, F


def mesh_config(cfg: int):
    """Mesh of BASELINE.json config cfg (1..5)."""
    v = L.dp(); f = L.u32p(); nv = C.c_uint64(); nf = C.c_uint64()
    L.check(L.host().p2m_mesh_config(cfg, C.byref(v), C.byref(nv), C.byref(f), C.byref(nf)))
    return _take_mesh(v, nv, f, nf)


def icosphere(level: int):
    v = L.dp(); f = L.u32p(); nv = C.c_uint64(); nf = C.c_uint64()
    L.check(L.host().p2m_mesh_icosphere(level, C.byref(v), C.byref(nv), C.byref(f), C.byref(nf)))
    return _take_mesh(v, nv, f, nf)


def gen_queries(cfg: int, vertices, faces, first: int, count: int, out: Optional[np.ndarray] = None):
    v, f = _as_mesh(vertices, faces)
    if out is None:
        out = np.empty((count, 3))
    L.check(L.host().p2m_gen_queries(cfg, L.ptr(v), len(v), L.ptr(f, L.u32p), len(f), first, count, L.ptr(out)))
    return out


def delaunay_adjacency(points):
    """Delaunay adjacency (CSR offsets, neighbours) of an arbitrary point set -- the DelaunayWalk
    graph (REF/SPEC.md:476), valid for queries inside 10x the points' AABB."""
    xyz = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    o = L.u64p(); a = L.u32p()
    L.check(L.host().p2m_delaunay_adjacency(L.ptr(xyz), len(xyz), C.byref(o), C.byref(a)))
    try:
        off = np.ctypeslib.as_array(o, shape=(len(xyz) + 1,)).copy()
        adj = np.ctypeslib.as_array(a, shape=(max(1, int(off[-1])),))[: int(off[-1])].copy()
    finally:
        L.host().p2m_free(C.cast(o, C.c_void_p))
        L.host().p2m_free(C.cast(a, C.c_void_p))
    return off, adj


def gen_uniform(seed: int, lo, hi, first: int, count: int):
    lo = np.ascontiguousarray(lo, dtype=np.float64); hi = np.ascontiguousarray(hi, dtype=np.float64)
    out = np.empty((count, 3))
    L.check(L.host().p2m_gen_uniform(seed, L.ptr(lo), L.ptr(hi), first, count, L.ptr(out)))
    return out
