// bvh.cpp -- see bvh.hpp.
#include "bvh.hpp"

#include <algorithm>

namespace p2m {

namespace {
struct Builder {
    Bvh* self;
    std::vector<BvhNode>& nodes;
    std::vector<uint32_t>& perm;
    const std::vector<V3>& cen;
    const double* tri;
    int leaf;

    uint32_t rec(uint32_t lo, uint32_t hi) {
        uint32_t me = (uint32_t)nodes.size();
        nodes.push_back(BvhNode{});
        Box b, cb;
        for (uint32_t i = lo; i < hi; ++i) {
            const double* t = tri + 9 * (uint64_t)perm[i];
            b.add(ld3(t)); b.add(ld3(t + 3)); b.add(ld3(t + 6));
            cb.add(cen[perm[i]]);
        }
        nodes[me].box = b;
        if ((int)(hi - lo) <= leaf) {
            nodes[me].first = lo; nodes[me].count = hi - lo; nodes[me].right = 0;
            return me;
        }
        V3 e = cb.ext();
        int ax = 0;
        if (e.y > comp(e, ax)) ax = 1;
        if (e.z > comp(e, ax)) ax = 2;
        uint32_t mid = lo + (hi - lo) / 2;
        std::nth_element(perm.begin() + lo, perm.begin() + mid, perm.begin() + hi,
                         [&](uint32_t x, uint32_t y) {
                             double cx = comp(cen[x], ax), cy = comp(cen[y], ax);
                             return cx < cy || (cx == cy && x < y);
                         });
        rec(lo, mid);                 // left child = me + 1
        uint32_t r = rec(mid, hi);
        nodes[me].right = r;
        nodes[me].count = 0;
        nodes[me].first = 0;
        return me;
    }
};
}  // namespace

void Bvh::build(const double* tri, uint64_t nf, int leaf_size) {
    tri_ = tri;
    nf_ = nf;
    nodes_.clear();
    perm_.resize(nf);
    for (uint64_t i = 0; i < nf; ++i) perm_[i] = (uint32_t)i;
    if (nf == 0) return;
    std::vector<V3> cen(nf);
    for (uint64_t f = 0; f < nf; ++f) cen[f] = (A(f) + B(f) + C(f)) * (1.0 / 3.0);
    nodes_.reserve(2 * nf / leaf_size + 4);
    Builder bd{this, nodes_, perm_, cen, tri, leaf_size};
    bd.rec(0, (uint32_t)nf);
}

uint32_t Bvh::closest(V3 q, double* d2out, V3* pout) const {
    double best = std::numeric_limits<double>::infinity();
    uint32_t bf = UINT32_MAX;
    V3 bp{0, 0, 0};
    if (nodes_.empty()) { *d2out = best; *pout = bp; return bf; }
    uint32_t st[128];
    int sp = 0;
    st[sp++] = 0;
    while (sp) {
        uint32_t n = st[--sp];
        const BvhNode& nd = nodes_[n];
        // visit when the box lower bound does not exceed the best (relative margin: a face whose
        // rounded closest point lands a few ulps outside its box is never skipped)
        if (nd.box.sqdist(q) > best * (1.0 + 1e-12)) continue;
        if (nd.count) {
            for (uint32_t i = nd.first; i < nd.first + nd.count; ++i) {
                uint32_t f = perm_[i];
                V3 p;
                double d2v = closest_tri(q, A(f), B(f), C(f), &p);
                if (d2v < best || (d2v == best && f < bf)) { best = d2v; bf = f; bp = p; }
            }
            continue;
        }
        uint32_t l = n + 1, r = nd.right;
        double dl = nodes_[l].box.sqdist(q), dr = nodes_[r].box.sqdist(q);
        if (dl <= dr) { st[sp++] = r; st[sp++] = l; }
        else { st[sp++] = l; st[sp++] = r; }
    }
    *d2out = best;
    *pout = bp;
    return bf;
}

namespace {
struct BallWalk {
    const Bvh& bvh;
    const Ball* balls;
    const double* tri;
    std::vector<uint32_t>& out;
    std::vector<uint8_t>& mark;

    void rec(uint32_t n, const std::vector<int>& act) {
        const BvhNode& nd = bvh.nodes()[n];
        if (nd.count) {
            for (uint32_t i = nd.first; i < nd.first + nd.count; ++i) {
                uint32_t f = bvh.perm()[i];
                if (mark[f]) continue;
                const double* t = tri + 9 * (uint64_t)f;
                V3 a = ld3(t), b = ld3(t + 3), c = ld3(t + 6);
                bool hit = false;
                for (int k : act) {
                    const Ball& bl = balls[k];
                    if (d2(a, bl.c) <= bl.r2 || d2(b, bl.c) <= bl.r2 || d2(c, bl.c) <= bl.r2) { hit = true; break; }
                    V3 p;
                    if (closest_tri(bl.c, a, b, c, &p) <= bl.r2) { hit = true; break; }
                }
                if (hit) { mark[f] = 1; out.push_back(f); }
            }
            return;
        }
        uint32_t kids[2] = {n + 1, nd.right};
        std::vector<int> sub;
        sub.reserve(act.size());
        for (uint32_t kid : kids) {
            sub.clear();
            const Box& cb = bvh.nodes()[kid].box;
            for (int k : act)
                if (cb.sqdist(balls[k].c) <= balls[k].r2) sub.push_back(k);
            if (!sub.empty()) rec(kid, sub);
        }
    }
};
}  // namespace

void Bvh::balls_query(const Ball* balls, int nballs, std::vector<uint32_t>& out,
                      std::vector<uint8_t>& mark) const {
    if (nodes_.empty() || nballs <= 0) return;
    std::vector<int> act;
    for (int k = 0; k < nballs; ++k)
        if (nodes_[0].box.sqdist(balls[k].c) <= balls[k].r2) act.push_back(k);
    size_t first_out = out.size();
    if (!act.empty()) {
        BallWalk w{*this, balls, tri_, out, mark};
        w.rec(0, act);
    }
    for (size_t i = first_out; i < out.size(); ++i) mark[out[i]] = 0;
}

}  // namespace p2m
