"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE's own code.

Run in the build container (needs oracle/_ref/libp2m_ref.so, compiled from
/root/reference/proj/src/geom.cpp by oracle/Makefile):

    python tests/golden/make_golden.py

Fixtures (small, committed):
  closest_tri.npz  -- 4096 seeded (q, a, b, c) cases incl. vertex/edge/face regions, near-degenerate
                      and far points -> p2mx::closest_on_triangle_sq d^2 and point (REF geom.cpp:31-70),
                      and p2mx::triangle_bounding_sphere of each (a, b, c) (REF geom.cpp:96-120)
  engine_ico2.npz  -- a built engine (icosphere level 2) + 3000 queries (uniform in 1.3x AABB, on
                      vertices, and outside D) -> the reference CPU query path (oracle/_ref: the
                      restated query loop calling p2mx::closest_on_triangle_sq), PRUNE_SAFE
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2605_00429_b200 as P  # noqa: E402


def closest_cases():
    rng = np.random.default_rng(20260601)
    n = 4096
    tri = rng.normal(size=(n, 3, 3)) * 10.0 ** rng.integers(-2, 3, size=(n, 1, 1))
    q = rng.normal(size=(n, 3)) * 3.0
    # region coverage: points near vertices, on edges, above faces, coplanar, far away
    for i in range(n):
        a, b, c = tri[i]
        k = i % 8
        if k == 1:
            q[i] = a + 1e-9 * rng.normal(size=3)
        elif k == 2:
            t = rng.uniform()
            q[i] = a + t * (b - a) + 1e-3 * rng.normal(size=3)
        elif k == 3:
            w = rng.dirichlet([1, 1, 1])
            nrm = np.cross(b - a, c - a)
            q[i] = w @ tri[i] + rng.normal() * nrm
        elif k == 4:
            w = rng.dirichlet([1, 1, 1]) * 1.5 - 0.25
            q[i] = w[0] * a + w[1] * b + (1 - w[0] - w[1]) * c
        elif k == 5:
            q[i] = q[i] * 1e6
        elif k == 6:
            tri[i, 2] = tri[i, 0] + (tri[i, 1] - tri[i, 0]) * 0.5 + 1e-7 * rng.normal(size=3)  # sliver
    d2 = np.zeros(n); p = np.zeros((n, 3)); sph = np.zeros((n, 4)); ok = np.zeros(n, bool)
    for i in range(n):
        d2[i], p[i] = O.closest_on_triangle_sq(q[i], *tri[i], reference=True)
        try:
            sph[i] = O.triangle_bounding_sphere(tri[i], reference=True)
            ok[i] = True
        except ValueError:
            sph[i] = np.nan
    np.savez_compressed(os.path.join(HERE, "closest_tri.npz"), q=q, tri=tri, d2=d2, p=p, sphere=sph, sphere_ok=ok)


def engine_case():
    V, F = P.icosphere(2)
    h = P.HostEngine.build(V, F)
    a = h.arrays()
    rng = np.random.default_rng(7)
    q = np.concatenate([rng.uniform(-1.3, 1.3, size=(2900, 3)), V[:80], [[40.0, 0, 0]] * 1,
                        rng.uniform(-30, 30, size=(19, 3))])
    ref = O.OracleEngine(a, reference=True).batch_query(q, prune=O.PRUNE_SAFE, per_query=True)
    np.savez_compressed(
        os.path.join(HERE, "engine_ico2.npz"),
        vertices=V, faces=F, site_xyz=a["site_xyz"], site_kind=a["site_kind"], tri=a["tri"],
        sphere=a["sphere"], list_offsets=a["list_offsets"], list_faces=a["list_faces"], domain=a["domain"],
        q=q, distance=ref["distance"], closest=ref["closest"], face=ref["face"], site=ref["site"],
        flags=ref["flags"], per_query=ref["per_query"])


if __name__ == "__main__":
    assert O.have_reference(), "oracle/_ref/libp2m_ref.so missing: run `make -C oracle` with /root/reference present"
    closest_cases()
    engine_case()
    print("golden fixtures written to", HERE)
