"""ctypes bindings of the C ABI in include/p2m.h (libp2m_host.so, libp2m_cuda.so).

The native libraries are built in-tree by `make` (see __graft_entry__.build()).  Loading fails
loudly: there is no Python or CPU fallback for the query path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(_HERE, "lib")
LIBDIR = os.environ.get("P2M_LIB_DIR", LIBDIR)  # A/B builds of the same sources (scripts/)

P2M_OK = 0
ERRORS = {
    -1: "P2M_ERR_INVALID",
    -2: "P2M_ERR_CUDA",
    -3: "P2M_ERR_NOT_BUILT",
    -4: "P2M_ERR_GEOMETRY",
    -5: "P2M_ERR_OOM",
    -6: "P2M_ERR_IO",
    -7: "P2M_ERR_INTERNAL",
}
SITE_MESH_VERTEX, SITE_SENTINEL, SITE_AUXILIARY = 0, 1, 2
FLAG_FALLBACK, FLAG_OUT_OF_DOMAIN, FLAG_TABLE_MISS = 1, 2, 4

dp = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class EngineDesc(C.Structure):
    _fields_ = [
        ("n_sites", C.c_uint64),
        ("site_xyz", dp),
        ("site_kind", u8p),
        ("n_faces", C.c_uint64),
        ("tri_xyz", dp),
        ("face_sphere", dp),
        ("list_offsets", u64p),
        ("list_faces", u32p),
        ("domain_min", C.c_double * 3),
        ("domain_max", C.c_double * 3),
        ("site_cell_box", dp),
        ("site_ref_xyz", dp),
        ("adj_offsets", u64p),
        ("adj_sites", u32p),
    ]


class Counters(C.Structure):
    _fields_ = [
        ("n_queries", C.c_uint64),
        ("candidates_visited", C.c_uint64),
        ("exact_evaluations", C.c_uint64),
        ("pruned", C.c_uint64),
        ("fallbacks", C.c_uint64),
        ("kd_nodes_visited", C.c_uint64),
        ("filter_passes", C.c_uint64),
        ("warp_rare_iters", C.c_uint64),
        ("structure_bytes", C.c_uint64),
        ("scan_tiles", C.c_uint64),
    ]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class BuildConfig(C.Structure):
    _fields_ = [
        ("augment", C.c_int),
        ("alpha", C.c_double),
        ("k", C.c_int),
        ("rho", C.c_double),
        ("max_rounds", C.c_int),
        ("domain_scale", C.c_double),
        ("n_threads", C.c_int),
        ("strict_mesh", C.c_int),
        ("aux_corner_union", C.c_int),
    ]


class BuildStats(C.Structure):
    _fields_ = [
        ("n_input_vertices", C.c_uint64),
        ("n_input_faces", C.c_uint64),
        ("n_vertices", C.c_uint64),
        ("n_faces", C.c_uint64),
        ("merged_vertices", C.c_uint64),
        ("removed_faces", C.c_uint64),
        ("n_sites", C.c_uint64),
        ("n_aux_sites", C.c_uint64),
        ("rounds_used", C.c_int),
        ("mean_edge", C.c_double),
        ("tau", C.c_double),
        ("list_entries", C.c_uint64),
        ("list_max", C.c_uint64),
        ("list_avg", C.c_double),
        ("t_voronoi_s", C.c_double),
        ("t_augment_s", C.c_double),
        ("t_tables_s", C.c_double),
        ("t_total_s", C.c_double),
        ("cell_corners", C.c_uint64),
    ]

    def as_dict(self):
        return {k: (getattr(self, k)) for k, _ in self._fields_}


class TableJob(C.Structure):
    """p2m_table_job (include/p2m.h)."""

    _fields_ = [
        ("n_sites", C.c_uint64),
        ("ball_off", u64p),
        ("balls", dp),
        ("n_faces", C.c_uint64),
        ("tri", dp),
        ("n_nodes", C.c_uint64),
        ("node_box", dp),
        ("node_meta", u32p),
        ("perm", u32p),
    ]


TABLE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, u64p, C.POINTER(u32p))


class P2MError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


_host = None
_cuda = None


def _load(name: str) -> C.CDLL:
    path = os.path.join(LIBDIR, name)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the native libraries first "
            "(python -c 'import __graft_entry__ as g; g.build()' or `make`)"
        )
    return C.CDLL(path, mode=C.RTLD_GLOBAL)


def host() -> C.CDLL:
    global _host
    if _host is None:
        L = _load("libp2m_host.so")
        L.p2m_last_error.restype = C.c_char_p
        L.p2m_build_config_default.argtypes = [C.POINTER(BuildConfig)]
        L.p2m_build.argtypes = [dp, C.c_uint64, u32p, C.c_uint64, C.POINTER(BuildConfig), C.POINTER(C.c_void_p)]
        L.p2m_build_with.argtypes = [dp, C.c_uint64, u32p, C.c_uint64, C.POINTER(BuildConfig), C.c_void_p,
                                     C.c_void_p, C.POINTER(C.c_void_p)]
        L.p2m_host_engine_destroy.argtypes = [C.c_void_p]
        L.p2m_host_engine_desc.argtypes = [C.c_void_p, C.POINTER(EngineDesc)]
        L.p2m_host_engine_stats.argtypes = [C.c_void_p, C.POINTER(BuildStats)]
        L.p2m_host_engine_mesh.argtypes = [C.c_void_p, C.POINTER(dp), u64p, C.POINTER(u32p), u64p]
        L.p2m_host_engine_site_refs.argtypes = [C.c_void_p, C.POINTER(dp)]
        L.p2m_host_engine_cell_corners.argtypes = [C.c_void_p, C.c_uint64, dp, C.c_uint64, u64p]
        L.p2m_host_closest_point.argtypes = [C.c_void_p, dp, dp, dp, u32p]
        L.p2m_host_engine_save.argtypes = [C.c_void_p, C.c_char_p]
        L.p2m_host_engine_load.argtypes = [C.c_char_p, dp, C.c_uint64, u32p, C.c_uint64, C.POINTER(C.c_void_p)]
        L.p2m_mesh_config.argtypes = [C.c_int, C.POINTER(dp), u64p, C.POINTER(u32p), u64p]
        L.p2m_mesh_icosphere.argtypes = [C.c_int, C.POINTER(dp), u64p, C.POINTER(u32p), u64p]
        L.p2m_gen_queries.argtypes = [C.c_int, dp, C.c_uint64, u32p, C.c_uint64, C.c_uint64, C.c_uint64, dp]
        L.p2m_gen_uniform.argtypes = [C.c_uint64, dp, dp, C.c_uint64, C.c_uint64, dp]
        L.p2m_free.argtypes = [C.c_void_p]
        L.p2m_delaunay_adjacency.argtypes = [dp, C.c_uint64, C.POINTER(u64p), C.POINTER(u32p)]
        _host = L
    return _host


def cuda() -> C.CDLL:
    """The device engine.  Raises if libp2m_cuda.so is absent -- never falls back."""
    global _cuda
    if _cuda is None:
        host()  # DT_NEEDED dependency, loaded first so the error string is shared
        L = _load("libp2m_cuda.so")
        vp = C.c_void_p
        L.p2m_engine_create.argtypes = [C.POINTER(EngineDesc), C.c_int, C.POINTER(C.c_int), C.POINTER(vp)]
        L.p2m_engine_destroy.argtypes = [vp]
        L.p2m_engine_save.argtypes = [vp, C.c_char_p]
        L.p2m_engine_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_int), C.POINTER(vp)]
        L.p2m_engine_info.argtypes = [vp, C.POINTER(C.c_int), dp, u64p]
        L.p2m_query.argtypes = [vp, dp, C.c_uint64, dp, dp, u32p, u32p, u32p, C.POINTER(Counters)]
        L.p2m_query_device.argtypes = [vp, C.c_int, vp, C.c_uint64, vp, vp, vp, vp, vp, vp, C.POINTER(Counters)]
        L.p2m_nearest_site_device.argtypes = [vp, C.c_int, vp, C.c_uint64, vp, vp]
        L.p2m_query_device_counters.argtypes = [vp, C.c_int, vp, C.c_uint64, vp, vp]
        L.p2m_set_profiling.argtypes = [vp, C.c_int]
        L.p2m_last_timings.argtypes = [vp, C.c_int, C.POINTER(C.c_float)]
        L.p2m_kernels_per_query.argtypes = [vp, C.c_uint64, C.POINTER(C.c_int)]
        L.p2m_set_scan_mode.argtypes = [vp, C.c_int]
        for name, at in (("p2m_set_nns_strategy", [vp, C.c_int]),
                         ("p2m_build_device", [dp, C.c_uint64, u32p, C.c_uint64, C.POINTER(BuildConfig), C.c_int,
                                               C.POINTER(vp)]),
                         ("p2m_table_job_device", [vp, vp, u64p, C.POINTER(u32p)])):
            if hasattr(L, name):  # absent only in A/B builds of older sources (scripts/gpu_ab.sh)
                getattr(L, name).argtypes = at
        _cuda = L
    return _cuda


def check(rc: int) -> None:
    if rc != P2M_OK:
        msg = host().p2m_last_error()
        raise P2MError(rc, msg.decode() if msg else "")


def ptr(a, t=dp):
    return a.ctypes.data_as(t)
