// p2m_traverse.cuh -- per-query tree traversals shared by the query kernels:
//   nearest_site  exact nearest site by the stack-free left-balanced k-d tree descent
//                 (REF/SPEC.md:482-487, ties -> lowest site id)
//   bvh_closest   exact closest point over all faces by the fallback BVH (REF/SPEC.md:201-209, 491)
#pragma once

#include "p2m_device.cuh"

namespace p2m {
namespace dev {

struct NN {
    double d2;
    uint32_t id;
    uint32_t visited;
    bool sentinel;
};

// Stack-free traversal of a left-balanced k-d tree (parent = (k+1)/2-1): the node visit order is
// exactly the recursive near-child-first order of the oracle (oracle/p2m_oracle.c nn_rec).
__device__ __forceinline__ NN nearest_site(const Params& p, V q) {
    NN r{__longlong_as_double(0x7ff0000000000000ll), 0xffffffffu, 0u, false};
    const int N = (int)p.n_nodes;
    int curr = 0, prev = -1;
    for (;;) {
        const int parent = ((curr + 1) >> 1) - 1;
        if (curr >= N) { prev = curr; curr = parent; continue; }
        const D4 nd = ldg4(p.kd + curr);
        const uint64_t meta = (uint64_t)__double_as_longlong(nd.w);
        const bool from_parent = prev < curr;
        if (from_parent) {
            const double dd = vd2(q, V{nd.x, nd.y, nd.z});
            const uint32_t id = (uint32_t)(meta & kIdMask);
            ++r.visited;
            if (dd < r.d2 || (dd == r.d2 && id < r.id)) { r.d2 = dd; r.id = id; r.sentinel = (meta & kSentinelBit) != 0; }
        }
        const int dim = (int)((meta >> kDimShift) & 3);
        const double diff = (dim == 0 ? q.x : (dim == 1 ? q.y : q.z)) - (dim == 0 ? nd.x : (dim == 1 ? nd.y : nd.z));
        const int right = diff > 0.0;
        const int close_c = 2 * curr + 1 + right;
        const int far_c = 2 * curr + 2 - right;
        int next;
        if (from_parent) next = close_c;
        else if (prev == close_c) next = (diff * diff <= r.d2) ? far_c : parent;
        else next = parent;
        if (next < 0) break;
        prev = curr;
        curr = next;
    }
    return r;
}

// nearest_site through the grid when q is inside the grid box: the exact lexicographic (d^2, id)
// minimum over every site whose Voronoi cell box meets q's grid cell -- a superset of the sites
// whose (closed) cell contains q, so it is the exact nearest site with lowest-id ties.  Falls back
// to the k-d tree outside the grid box or when the engine has no grid.
__device__ __forceinline__ NN nearest_site_cl(const Params& p, V q) {
    uint32_t c;
    if (!p.grid_off || !grid_cell(p, q, &c)) return nearest_site(p, q);
    NN r{__longlong_as_double(0x7ff0000000000000ll), 0xffffffffu, 0u, false};
    const uint32_t b = p.grid_off[c], e = p.grid_off[c + 1];
    if (b == e) return nearest_site(p, q);
    for (uint32_t j = b; j < e; ++j) {
        const uint32_t id = p.grid_site[j];
        const D4 s = ldg4(p.site_pos + id);
        const double dd = vd2(q, V{s.x, s.y, s.z});
        ++r.visited;
        if (dd < r.d2 || (dd == r.d2 && id < r.id)) {
            r.d2 = dd;
            r.id = id;
            r.sentinel = ((uint64_t)__double_as_longlong(s.w) & kSentinelBit) != 0;
        }
    }
    return r;
}

// DelaunayWalk nearest_site (REF/SPEC.md:476, 516; oracle/p2m_oracle.c orc_walk_nearest): greedy
// descent on the Delaunay adjacency -- move to the neighbour with the smallest (d^2, id) while it
// beats the current site -- warm-started from the first site listed in q's grid cell (site 0
// outside the grid box).  If the final site has an exactly equidistant neighbour, the tie set is
// flooded and its lowest id returned (up to 16 tied sites; beyond that the k-d tree answers).
__device__ __forceinline__ NN nearest_site_walk(const Params& p, V q) {
    uint32_t v = 0, c;
    if (p.grid_off && grid_cell(p, q, &c)) {
        const uint32_t b = p.grid_off[c];
        if (b < p.grid_off[c + 1]) v = p.grid_site[b];
    }
    D4 sv = ldg4(p.site_pos + v);
    double dv = vd2(q, V{sv.x, sv.y, sv.z});
    uint32_t visited = 1;
    bool tie = false;
    for (;;) {
        uint32_t bst = v;
        double bd = dv;
        tie = false;
        const uint64_t k1 = p.adj_off[v + 1];
        for (uint64_t k = p.adj_off[v]; k < k1; ++k) {
            const uint32_t w = p.adj[k];
            const D4 s = ldg4(p.site_pos + w);
            const double d = vd2(q, V{s.x, s.y, s.z});
            ++visited;
            tie |= d == dv;
            if (d < bd || (d == bd && w < bst)) { bst = w; bd = d; }
        }
        if (bst == v) break;
        v = bst;
        dv = bd;
    }
    uint32_t best = v;
    if (tie) {
        uint32_t set[16];
        int n = 1, head = 0;
        set[0] = v;
        while (head < n) {
            const uint32_t u = set[head++];
            for (uint64_t k = p.adj_off[u]; k < p.adj_off[u + 1]; ++k) {
                const uint32_t w = p.adj[k];
                const D4 s = ldg4(p.site_pos + w);
                ++visited;
                if (vd2(q, V{s.x, s.y, s.z}) != dv) continue;
                bool seen = false;
                for (int i = 0; i < n; ++i) seen |= set[i] == w;
                if (seen) continue;
                if (n == 16) {
                    NN r = nearest_site(p, q);
                    r.visited += visited;
                    return r;
                }
                set[n++] = w;
                best = min(best, w);
            }
        }
        sv = ldg4(p.site_pos + best);
    } else {
        sv = ldg4(p.site_pos + best);
    }
    NN r;
    r.d2 = dv;
    r.id = best;
    r.visited = visited;
    r.sentinel = ((uint64_t)__double_as_longlong(sv.w) & kSentinelBit) != 0;
    return r;
}

// the engine's nearest_site strategy (P2M_NNS_*, include/p2m.h)
__device__ __forceinline__ NN nearest_site_any(const Params& p, V q) {
    if (p.nns == 2 && p.adj_off) return nearest_site_walk(p, q);
    if (p.nns == 1) return nearest_site(p, q);
    return nearest_site_cl(p, q);
}

// Exact global closest point by the fallback BVH (REF/SPEC.md:201-209, 491): lowest face id on
// exact d^2 ties; a node is skipped only when its box is farther than best*(1+1e-12).
__device__ __forceinline__ uint32_t bvh_closest(const Params& p, V q, double* best_out) {
    double best = __longlong_as_double(0x7ff0000000000000ll);
    uint32_t bf = 0xffffffffu;
    uint32_t st[64];
    int sp = 0;
    st[sp++] = 0;
    while (sp) {
        const uint32_t n = st[--sp];
        const D4 b0 = ldg4(p.bvh + 2 * (uint64_t)n), b1 = ldg4(p.bvh + 2 * (uint64_t)n + 1);
        auto boxd = [&](const D4& x0, const D4& x1) {
            const double lo[3] = {x0.x, x0.y, x0.z}, hi[3] = {x0.w, x1.x, x1.y}, v[3] = {q.x, q.y, q.z};
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if (v[k] < lo[k]) s += (lo[k] - v[k]) * (lo[k] - v[k]);
                else if (v[k] > hi[k]) s += (v[k] - hi[k]) * (v[k] - hi[k]);
            }
            return s;
        };
        if (boxd(b0, b1) > best * (1.0 + 1e-12)) continue;
        const uint64_t meta = (uint64_t)__double_as_longlong(b1.z);
        const uint32_t cnt = (uint32_t)(meta >> 32), idx = (uint32_t)meta;
        if (cnt) {
            for (uint32_t i = idx; i < idx + cnt; ++i) {
                const uint32_t f = p.bvh_perm[i];
                V a, b, c, pp;
                load_tri(p.rec + 4 * (uint64_t)f, &a, &b, &c);
                const double dd = closest_tri(q, a, b, c, &pp);
                if (dd < best || (dd == best && f < bf)) { best = dd; bf = f; }
            }
            continue;
        }
        const uint32_t l = n + 1, r = idx;
        const double dl = boxd(ldg4(p.bvh + 2 * (uint64_t)l), ldg4(p.bvh + 2 * (uint64_t)l + 1));
        const double dr = boxd(ldg4(p.bvh + 2 * (uint64_t)r), ldg4(p.bvh + 2 * (uint64_t)r + 1));
        if (sp + 2 > 64) break;  // depth is bounded by ~2 log2(F) for median splits
        if (dl <= dr) { st[sp++] = r; st[sp++] = l; }
        else { st[sp++] = l; st[sp++] = r; }
    }
    *best_out = best;
    return bf;
}

}  // namespace dev
}  // namespace p2m
