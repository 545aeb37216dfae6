// ref_shim.cpp -- extern "C" wrappers over the reference's own geometry primitives
// (TEST INFRASTRUCTURE ONLY).  Compiled together with REF/proj/src/geom.cpp, where it lies under
// /root/reference, into oracle/_ref/libp2m_ref.so by oracle/Makefile.  Nothing here restates the
// reference: every function forwards to p2mx:: unchanged so the tests can pin the oracle
// restatement (oracle/p2m_oracle.c) and the product's host builder against the real thing.
#include "p2mx/geom.hpp"

#include <cstdint>

using p2mx::Vec3;

static inline Vec3 v3(const double* p) { return Vec3{p[0], p[1], p[2]}; }

extern "C" {

// REF/proj/src/geom.cpp:31-70
__attribute__((visibility("default"))) void p2mref_closest_on_triangle_sq(
    const double* q, const double* a, const double* b, const double* c, double* d2, double* p) {
    p2mx::ClosestPoint r = p2mx::closest_on_triangle_sq(v3(q), v3(a), v3(b), v3(c));
    *d2 = r.distance;
    p[0] = r.point.x; p[1] = r.point.y; p[2] = r.point.z;
}

// REF/proj/src/geom.cpp:82-88; returns 0 on success, -4 on GeometryError
__attribute__((visibility("default"))) int p2mref_point_triangle_distance(
    const double* q, const double* t, double* dist, double* p) {
    try {
        p2mx::ClosestPoint r =
            p2mx::point_triangle_distance(v3(q), p2mx::Triangle3{v3(t), v3(t + 3), v3(t + 6)});
        *dist = r.distance;
        p[0] = r.point.x; p[1] = r.point.y; p[2] = r.point.z;
        return 0;
    } catch (const p2mx::GeometryError&) {
        return -4;
    }
}

// REF/proj/src/geom.cpp:90-94
__attribute__((visibility("default"))) int p2mref_sphere_triangle_intersect(const double* s4,
                                                                            const double* t) {
    try {
        return p2mx::sphere_triangle_intersect(p2mx::Sphere{v3(s4), s4[3]},
                                               p2mx::Triangle3{v3(t), v3(t + 3), v3(t + 6)})
                   ? 1
                   : 0;
    } catch (const p2mx::GeometryError&) {
        return -4;
    }
}

// REF/proj/src/geom.cpp:96-120
__attribute__((visibility("default"))) int p2mref_triangle_bounding_sphere(const double* t,
                                                                           double* out4) {
    try {
        p2mx::Sphere s =
            p2mx::triangle_bounding_sphere(p2mx::Triangle3{v3(t), v3(t + 3), v3(t + 6)});
        out4[0] = s.center.x; out4[1] = s.center.y; out4[2] = s.center.z; out4[3] = s.radius;
        return 0;
    } catch (const p2mx::GeometryError&) {
        return -4;
    }
}

// REF/proj/src/geom.cpp:282-321 (throwing variant); 0 ok, -4 coplanar
__attribute__((visibility("default"))) int p2mref_tetra_circumcenter(const double* p0,
                                                                     const double* p1,
                                                                     const double* p2,
                                                                     const double* p3,
                                                                     double* out) {
    try {
        Vec3 c = p2mx::tetra_circumcenter(v3(p0), v3(p1), v3(p2), v3(p3));
        out[0] = c.x; out[1] = c.y; out[2] = c.z;
        return 0;
    } catch (const p2mx::GeometryError&) {
        return -4;
    }
}

// REF/proj/src/geom.cpp:219-225, 272-278
__attribute__((visibility("default"))) int p2mref_orient3d(const double* a, const double* b,
                                                           const double* c, const double* d) {
    return p2mx::orient3d(v3(a), v3(b), v3(c), v3(d));
}
__attribute__((visibility("default"))) int p2mref_in_sphere(const double* a, const double* b,
                                                            const double* c, const double* d,
                                                            const double* e) {
    return p2mx::in_sphere(v3(a), v3(b), v3(c), v3(d), v3(e));
}

// REF/proj/src/geom.cpp:7-19
__attribute__((visibility("default"))) void p2mref_aabb_scaled(const double* mn, const double* mx,
                                                               double factor, double min_frac,
                                                               double* out6) {
    p2mx::Aabb b{v3(mn), v3(mx)};
    p2mx::Aabb s = b.scaled_about_center(factor, min_frac);
    out6[0] = s.min.x; out6[1] = s.min.y; out6[2] = s.min.z;
    out6[3] = s.max.x; out6[4] = s.max.y; out6[5] = s.max.z;
}

}  // extern "C"
