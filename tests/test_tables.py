"""build_all_tables as a job (REF/SPEC.md:397-423, ball enumeration REF/SPEC.md:192-200;
SURVEY.md 8(f) row 3).

The builder hands the table phase to an executor through p2m_table_job (include/p2m.h).  Three
executors must give the same CSR bit for bit:
  * the builder's own host threads (p2m_build),
  * a pure-Python walk below that restates the job contract with Python floats (IEEE fp64, no
    contraction, same operation order) -- this pins the contract on CPU,
  * the GPU executor p2m_build_device / p2m_table_job_device (`-m gpu`).
"""
import numpy as np
import pytest

import paper_2605_00429_b200 as P
from paper_2605_00429_b200 import _lib as L

from test_builder import TET_F, TET_V, bumpy_sphere


def _d2(p, q):
    dx, dy, dz = p[0] - q[0], p[1] - q[1], p[2] - q[2]
    return dx * dx + dy * dy + dz * dz


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _axpy(a, d, s):
    return (a[0] + d[0] * s, a[1] + d[1] * s, a[2] + d[2] * s)


def closest_tri_sq(q, a, b, c):
    """REF/proj/src/geom.cpp:31-70 in Python floats (same operation order as geom.hpp)."""
    ab, ac, aq = _sub(b, a), _sub(c, a), _sub(q, a)
    s1, s2 = _dot(ab, aq), _dot(ac, aq)
    if s1 <= 0.0 and s2 <= 0.0:
        return _d2(q, a)
    bq = _sub(q, b)
    s3, s4 = _dot(ab, bq), _dot(ac, bq)
    if s3 >= 0.0 and s4 <= s3:
        return _d2(q, b)
    wc = s1 * s4 - s3 * s2
    if wc <= 0.0 and s1 >= 0.0 and s3 <= 0.0:
        return _d2(q, _axpy(a, ab, s1 / (s1 - s3)))
    cq = _sub(q, c)
    s5, s6 = _dot(ab, cq), _dot(ac, cq)
    if s6 >= 0.0 and s5 <= s6:
        return _d2(q, c)
    wb = s5 * s2 - s1 * s6
    if wb <= 0.0 and s2 >= 0.0 and s6 <= 0.0:
        return _d2(q, _axpy(a, ac, s2 / (s2 - s6)))
    wa = s3 * s6 - s5 * s4
    if wa <= 0.0 and (s4 - s3) >= 0.0 and (s5 - s6) >= 0.0:
        return _d2(q, _axpy(b, _sub(c, b), (s4 - s3) / ((s4 - s3) + (s5 - s6))))
    inv = 1.0 / (wa + wb + wc)
    return _d2(q, _axpy(_axpy(a, ab, wb * inv), ac, wc * inv))


def box_sqdist(box, p):
    s = 0.0
    for k in range(3):
        v, lo, hi = p[k], box[k], box[3 + k]
        if v < lo:
            s += (lo - v) * (lo - v)
        elif v > hi:
            s += (v - hi) * (v - hi)
    return s


def python_table_executor(job):
    """The job contract, literally: per ball, walk the BVH from the root with the box test, test
    every leaf face (vertex within r2, or closest_tri <= r2); lists = sorted union per site."""
    boff, balls, tri = job["ball_off"], job["balls"].tolist(), job["tri"].tolist()
    nbox, nmeta, perm = job["node_box"].tolist(), job["node_meta"].tolist(), job["perm"].tolist()
    S = len(boff) - 1
    off = np.zeros(S + 1, np.uint64)
    lists = []
    for s in range(S):
        hit = set()
        for b in range(int(boff[s]), int(boff[s + 1])):
            cx, cy, cz, r2 = balls[b]
            c = (cx, cy, cz)
            if not nbox or box_sqdist(nbox[0], c) > r2:
                continue
            stack = [0]
            while stack:
                n = stack.pop()
                right, first, count = nmeta[n]
                if count:
                    for k in range(first, first + count):
                        f = perm[k]
                        if f in hit:
                            continue
                        t = tri[f]
                        a, bb, cc = tuple(t[0:3]), tuple(t[3:6]), tuple(t[6:9])
                        if (_d2(a, c) <= r2 or _d2(bb, c) <= r2 or _d2(cc, c) <= r2
                                or closest_tri_sq(c, a, bb, cc) <= r2):
                            hit.add(f)
                    continue
                for kid in (n + 1, right):
                    if box_sqdist(nbox[kid], c) <= r2:
                        stack.append(kid)
        lst = sorted(hit)
        lists.extend(lst)
        off[s + 1] = off[s] + len(lst)
    return off, np.array(lists, np.uint32)


def _same_engine(h1, h2):
    a, b = h1.arrays(), h2.arrays()
    for k in ("site_xyz", "site_kind", "tri", "sphere", "list_offsets", "list_faces", "domain"):
        assert a[k].tobytes() == b[k].tobytes(), k


@pytest.mark.parametrize("mesh", ["tet", "ico2", "bumpy2"])
def test_table_job_python_executor_matches_host(mesh):
    V, F = {"tet": (TET_V, TET_F), "ico2": P.icosphere(2), "bumpy2": bumpy_sphere(level=2)}[mesh]
    h_host = P.HostEngine.build(V, F)
    h_job = P.HostEngine.build_with(V, F, python_table_executor)
    _same_engine(h_host, h_job)
    st = h_job.stats()
    assert st["list_entries"] == h_host.stats()["list_entries"]


def test_table_job_contract_arrays():
    V, F = P.icosphere(1)
    seen = {}

    def spy(job):
        seen.update(job)
        return python_table_executor(job)

    h = P.HostEngine.build_with(V, F, spy)
    a = h.arrays()
    S = len(a["site_xyz"])
    assert len(seen["ball_off"]) == S + 1 and seen["ball_off"][0] == 0
    kinds = a["site_kind"]
    nb = np.diff(seen["ball_off"].astype(np.int64))
    assert np.all(nb[kinds == L.SITE_SENTINEL] == 0)      # empty sentinel lists (REF/SPEC.md:418)
    assert np.all(nb[kinds != L.SITE_SENTINEL] >= 4)      # a bounded cell has >= 4 corners
    assert np.all(seen["balls"][:, 3] > 0)
    assert seen["tri"].tobytes() == a["tri"].reshape(-1, 9).tobytes()
    assert sorted(seen["perm"].tolist()) == list(range(len(F)))
    leaves = seen["node_meta"][seen["node_meta"][:, 2] > 0]
    assert leaves[:, 2].sum() == len(F) and leaves[:, 2].max() <= 4  # leaf size 4 (REF/SPEC.md:216)


def test_table_job_errors_propagate():
    V, F = P.icosphere(1)

    def broken(job):
        raise ValueError("executor exploded")

    with pytest.raises(ValueError, match="executor exploded"):
        P.HostEngine.build_with(V, F, broken)

    def bad_offsets(job):
        S = len(job["ball_off"]) - 1
        off = np.zeros(S + 1, np.uint64)
        off[1] = 5
        return off, np.zeros(5, np.uint32)

    with pytest.raises(L.P2MError, match="bad offsets"):
        P.HostEngine.build_with(V, F, bad_offsets)


# ---------------------------------------------------------------------------------------------
# GPU executor


def _gpu_vs_host(V, F, cfg=None):
    h_host = P.HostEngine.build(V, F, cfg)
    h_dev = P.HostEngine.build(V, F, cfg, table_device=0)
    _same_engine(h_host, h_dev)
    return h_host, h_dev


@pytest.mark.gpu
@pytest.mark.parametrize("mesh", ["tet", "ico3", "bumpy3", "c1", "c2"])
def test_gpu_tables_bit_identical(mesh):
    V, F = {"tet": (TET_V, TET_F), "ico3": P.icosphere(3), "bumpy3": bumpy_sphere(),
            "c1": P.mesh_config(1), "c2": P.mesh_config(2)}[mesh]
    h_host, h_dev = _gpu_vs_host(V, F)
    assert h_dev.stats()["list_entries"] > 0


@pytest.mark.gpu
def test_gpu_tables_spec_ball_option():
    V, F = bumpy_sphere()
    _gpu_vs_host(V, F, P.BuildConfig(aux_corner_union=False))


@pytest.mark.gpu
def test_gpu_table_job_python_contract():
    """The GPU executor and the pure-Python restatement agree on the same job."""
    V, F = bumpy_sphere(level=2)
    h_py = P.HostEngine.build_with(V, F, python_table_executor)
    h_dev = P.HostEngine.build(V, F, table_device=0)
    _same_engine(h_py, h_dev)


@pytest.mark.gpu
@pytest.mark.slow
def test_gpu_tables_c3():
    V, F = P.mesh_config(3)
    h_host, h_dev = _gpu_vs_host(V, F)
    st_h, st_d = h_host.stats(), h_dev.stats()
    print("c3 tables host %.2f s, gpu %.2f s" % (st_h["t_tables_s"], st_d["t_tables_s"]))
