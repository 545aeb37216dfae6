// geom.hpp -- fp64 geometry used by the host builder (product code, host side).
//
// The point-triangle kernel and the minimal bounding sphere restate the reference's
// REF/proj/src/geom.cpp:31-70 and :96-120 with the same operation order, so the spheres the
// builder uploads are bit-identical to p2mx::triangle_bounding_sphere (pinned by
// tests/test_builder.py against oracle/_ref).  Compiled with -ffp-contract=off.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>

namespace p2m {

struct V3 {
    double x, y, z;
};

inline V3 mk(double x, double y, double z) { return V3{x, y, z}; }
inline V3 ld3(const double* p) { return V3{p[0], p[1], p[2]}; }
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double sq(V3 a) { return dot(a, a); }
inline double d2(V3 a, V3 b) { return sq(a - b); }
inline double len(V3 a) { return std::sqrt(sq(a)); }
inline double comp(V3 a, int k) { return k == 0 ? a.x : (k == 1 ? a.y : a.z); }

struct Box {
    V3 lo{std::numeric_limits<double>::max(), std::numeric_limits<double>::max(),
          std::numeric_limits<double>::max()};
    V3 hi{std::numeric_limits<double>::lowest(), std::numeric_limits<double>::lowest(),
          std::numeric_limits<double>::lowest()};
    void add(V3 p) {
        lo.x = std::min(lo.x, p.x); lo.y = std::min(lo.y, p.y); lo.z = std::min(lo.z, p.z);
        hi.x = std::max(hi.x, p.x); hi.y = std::max(hi.y, p.y); hi.z = std::max(hi.z, p.z);
    }
    void add(const Box& b) { add(b.lo); add(b.hi); }
    V3 center() const { return (lo + hi) * 0.5; }
    V3 ext() const { return hi - lo; }
    double diag() const { return std::sqrt(d2(hi, lo)); }
    // squared distance from p to the box, 0 inside (REF geom.hpp:72-80)
    double sqdist(V3 p) const {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) {
            double v = comp(p, k), l = comp(lo, k), h = comp(hi, k);
            if (v < l) s += (l - v) * (l - v);
            else if (v > h) s += (v - h) * (v - h);
        }
        return s;
    }
    bool contains(V3 p) const {
        return p.x >= lo.x && p.x <= hi.x && p.y >= lo.y && p.y <= hi.y && p.z >= lo.z && p.z <= hi.z;
    }
    // extents scaled by f about the centre, flat axes padded to min_frac of the largest
    // (same definition as REF geom.cpp:7-19)
    Box scaled(double f, double min_frac) const {
        V3 c = center();
        V3 h = ext() * (0.5 * f);
        double fl = 0.0;
        if (min_frac > 0.0) {
            fl = min_frac * std::max({h.x, h.y, h.z});
            if (fl <= 0.0) fl = min_frac;
        }
        h.x = std::max(h.x, fl); h.y = std::max(h.y, fl); h.z = std::max(h.z, fl);
        Box b; b.lo = c - h; b.hi = c + h;
        return b;
    }
};

// closest point on triangle (a,b,c) to q; returns squared distance (REF geom.cpp:31-70)
inline double closest_tri(V3 q, V3 a, V3 b, V3 c, V3* pout) {
    const V3 ab = b - a, ac = c - a, aq = q - a;
    const double s1 = dot(ab, aq), s2 = dot(ac, aq);
    if (s1 <= 0.0 && s2 <= 0.0) { *pout = a; return d2(q, a); }
    const V3 bq = q - b;
    const double s3 = dot(ab, bq), s4 = dot(ac, bq);
    if (s3 >= 0.0 && s4 <= s3) { *pout = b; return d2(q, b); }
    const double wc = s1 * s4 - s3 * s2;
    if (wc <= 0.0 && s1 >= 0.0 && s3 <= 0.0) {
        const double t = s1 / (s1 - s3);
        *pout = a + ab * t; return d2(q, *pout);
    }
    const V3 cq = q - c;
    const double s5 = dot(ab, cq), s6 = dot(ac, cq);
    if (s6 >= 0.0 && s5 <= s6) { *pout = c; return d2(q, c); }
    const double wb = s5 * s2 - s1 * s6;
    if (wb <= 0.0 && s2 >= 0.0 && s6 <= 0.0) {
        const double t = s2 / (s2 - s6);
        *pout = a + ac * t; return d2(q, *pout);
    }
    const double wa = s3 * s6 - s5 * s4;
    if (wa <= 0.0 && (s4 - s3) >= 0.0 && (s5 - s6) >= 0.0) {
        const double t = (s4 - s3) / ((s4 - s3) + (s5 - s6));
        *pout = b + (c - b) * t; return d2(q, *pout);
    }
    const double inv = 1.0 / (wa + wb + wc);
    const double bv = wb * inv, bw = wc * inv;
    *pout = a + ab * bv + ac * bw;
    return d2(q, *pout);
}

// zero-area test of REF geom.cpp:76-80 (also catches NaN / coincident vertices)
inline bool tri_degenerate(V3 a, V3 b, V3 c) {
    const double s2 = std::max({d2(a, b), d2(a, c), d2(b, c)});
    const double cr2 = sq(cross(b - a, c - a));
    return !(cr2 > s2 * s2 * 1e-28);
}

// minimal enclosing sphere of a triangle (REF geom.cpp:96-120); out = cx, cy, cz, r
inline void tri_sphere(V3 a, V3 b, V3 c, double* out) {
    const V3 *P = &a, *Q = &b, *R = &c;
    const double lab = d2(a, b), lac = d2(a, c), lbc = d2(b, c);
    if (lac >= lab && lac >= lbc) { Q = &c; R = &b; }
    else if (lbc >= lab && lbc >= lac) { P = &b; Q = &c; R = &a; }
    const V3 m = (*P + *Q) * 0.5;
    const double r2 = d2(*P, *Q) * 0.25;
    if (d2(*R, m) <= r2) { out[0] = m.x; out[1] = m.y; out[2] = m.z; out[3] = std::sqrt(r2); return; }
    const V3 u = b - a, v = c - a;
    const double uu = dot(u, u), vv = dot(v, v), uv = dot(u, v);
    const double den = 2.0 * (uu * vv - uv * uv);
    const double s = (vv * (uu - uv)) / den;
    const double w = (uu * (vv - uv)) / den;
    const V3 cc = a + u * s + v * w;
    const double rr = std::max({d2(cc, a), d2(cc, b), d2(cc, c)});
    out[0] = cc.x; out[1] = cc.y; out[2] = cc.z; out[3] = std::sqrt(rr);
}

}  // namespace p2m
