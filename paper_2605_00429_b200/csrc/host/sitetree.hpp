// sitetree.hpp -- build-time k-d tree over site positions (bucketed leaves), for the Voronoi cell
// construction: k nearest neighbours of a site and "is any site strictly closer to corner u than
// the owning site" (the empty-ball certificate of a cell corner).  Not the query-time tree: the
// device's nearest-site tree is the left-balanced BFS tree packed by the CUDA library.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "geom.hpp"

namespace p2m {

class SiteTree {
   public:
    void build(const std::vector<V3>& pts, int leaf = 8) {
        pts_ = &pts;
        idx_.resize(pts.size());
        for (size_t i = 0; i < pts.size(); ++i) idx_[i] = (uint32_t)i;
        nodes_.clear();
        if (!pts.empty()) rec(0, (uint32_t)pts.size(), leaf);
    }

    // nearest site to q among those with d^2 < bound2 (strict); returns UINT32_MAX if none.
    // Ties on d^2 resolve to the lower id.
    uint32_t nearest(V3 q, double bound2, double* d2out) const {
        uint32_t best = UINT32_MAX;
        double bd = bound2;
        if (!nodes_.empty()) nn(0, q, bd, best, true);
        if (d2out) *d2out = bd;
        return best;
    }

    // k nearest to q (excluding id `skip`), ascending (d^2, id)
    void knn(V3 q, int k, uint32_t skip, std::vector<std::pair<double, uint32_t>>& out) const {
        out.clear();
        if (nodes_.empty() || k <= 0) return;
        knn_rec(0, q, k, skip, out);
        std::sort(out.begin(), out.end());
    }

   private:
    struct Node {
        Box box;
        uint32_t lo, hi;     // point range (leaf) or 0
        uint32_t left, right;
        bool leaf;
    };
    const std::vector<V3>* pts_ = nullptr;
    std::vector<uint32_t> idx_;
    std::vector<Node> nodes_;

    uint32_t rec(uint32_t lo, uint32_t hi, int leaf) {
        uint32_t me = (uint32_t)nodes_.size();
        nodes_.push_back(Node{});
        Box b;
        for (uint32_t i = lo; i < hi; ++i) b.add((*pts_)[idx_[i]]);
        nodes_[me].box = b;
        if ((int)(hi - lo) <= leaf) {
            nodes_[me].leaf = true; nodes_[me].lo = lo; nodes_[me].hi = hi;
            return me;
        }
        V3 e = b.ext();
        int ax = 0;
        if (e.y > comp(e, ax)) ax = 1;
        if (e.z > comp(e, ax)) ax = 2;
        uint32_t mid = lo + (hi - lo) / 2;
        const auto& P = *pts_;
        std::nth_element(idx_.begin() + lo, idx_.begin() + mid, idx_.begin() + hi,
                         [&](uint32_t x, uint32_t y) {
                             double a = comp(P[x], ax), c = comp(P[y], ax);
                             return a < c || (a == c && x < y);
                         });
        uint32_t l = rec(lo, mid, leaf);
        uint32_t r = rec(mid, hi, leaf);
        nodes_[me].leaf = false; nodes_[me].left = l; nodes_[me].right = r;
        return me;
    }

    void nn(uint32_t n, V3 q, double& bd, uint32_t& best, bool) const {
        const Node& nd = nodes_[n];
        if (nd.leaf) {
            for (uint32_t i = nd.lo; i < nd.hi; ++i) {
                uint32_t id = idx_[i];
                double dd = d2(q, (*pts_)[id]);
                if (dd < bd || (dd == bd && best != UINT32_MAX && id < best)) { bd = dd; best = id; }
            }
            return;
        }
        double dl = nodes_[nd.left].box.sqdist(q), dr = nodes_[nd.right].box.sqdist(q);
        if (dl <= dr) {
            if (dl <= bd) nn(nd.left, q, bd, best, true);
            if (dr <= bd) nn(nd.right, q, bd, best, true);
        } else {
            if (dr <= bd) nn(nd.right, q, bd, best, true);
            if (dl <= bd) nn(nd.left, q, bd, best, true);
        }
    }

    void knn_rec(uint32_t n, V3 q, int k, uint32_t skip, std::vector<std::pair<double, uint32_t>>& heap_) const {
        const Node& nd = nodes_[n];
        auto worst = [&]() { return (int)heap_.size() < k ? std::numeric_limits<double>::infinity() : heap_.front().first; };
        if (nd.leaf) {
            for (uint32_t i = nd.lo; i < nd.hi; ++i) {
                uint32_t id = idx_[i];
                if (id == skip) continue;
                std::pair<double, uint32_t> c{d2(q, (*pts_)[id]), id};
                if ((int)heap_.size() < k) {
                    heap_.push_back(c);
                    std::push_heap(heap_.begin(), heap_.end());
                } else if (c < heap_.front()) {
                    std::pop_heap(heap_.begin(), heap_.end());
                    heap_.back() = c;
                    std::push_heap(heap_.begin(), heap_.end());
                }
            }
            return;
        }
        double dl = nodes_[nd.left].box.sqdist(q), dr = nodes_[nd.right].box.sqdist(q);
        if (dl <= dr) {
            if (dl <= worst()) knn_rec(nd.left, q, k, skip, heap_);
            if (dr <= worst()) knn_rec(nd.right, q, k, skip, heap_);
        } else {
            if (dr <= worst()) knn_rec(nd.right, q, k, skip, heap_);
            if (dl <= worst()) knn_rec(nd.left, q, k, skip, heap_);
        }
    }
};

}  // namespace p2m
