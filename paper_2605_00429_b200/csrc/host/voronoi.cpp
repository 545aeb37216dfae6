// voronoi.cpp -- see voronoi.hpp.
#include "voronoi.hpp"

#include <algorithm>
#include <cmath>

namespace p2m {

void CellClipper::init_box(V3 v) {
    P_.clear(); ok_.clear(); fo_.clear(); fv_.clear(); fn_.clear();
    const V3 lo = outer_.lo - v, hi = outer_.hi - v;
    for (int i = 0; i < 8; ++i) {
        P_.push_back(V3{(i & 1) ? hi.x : lo.x, (i & 2) ? hi.y : lo.y, (i & 4) ? hi.z : lo.z});
        ok_.push_back(0);
    }
    static const int kF[6][4] = {{0, 4, 6, 2}, {1, 3, 7, 5}, {0, 1, 5, 4},
                                 {2, 6, 7, 3}, {0, 2, 3, 1}, {4, 5, 7, 6}};
    fo_.push_back(0);
    for (int f = 0; f < 6; ++f) {
        for (int k = 0; k < 4; ++k) fv_.push_back(kF[f][k]);
        fo_.push_back((int)fv_.size());
        fn_.push_back(-1 - f);
    }
}

// Keep {x : n.x <= d}.  Vertices within eps (distance) of the plane are kept as on-plane.
bool CellClipper::clip(V3 n, double d, int nb) {
    const double nl = len(n);
    const double tol = eps_ * nl;
    const int nv = (int)P_.size();
    s_.resize(nv);
    bool any = false;
    for (int i = 0; i < nv; ++i) {
        s_[i] = dot(P_[i], n) - d;
        if (s_[i] > tol) any = true;
    }
    if (!any) return false;
    ++clips_;
    map_.assign(nv, -1);
    nP_.clear(); nok_.clear();
    for (int i = 0; i < nv; ++i)
        if (s_[i] <= tol) { map_[i] = (int)nP_.size(); nP_.push_back(P_[i]); nok_.push_back(ok_[i]); }
    const int n_kept = (int)nP_.size();
    hits_.clear();
    auto edge_point = [&](int a, int b) -> int {  // a strictly inside, b strictly outside
        for (const EdgeHit& h : hits_)
            if (h.a == a && h.b == b) return h.id;
        const double t = s_[a] / (s_[a] - s_[b]);
        V3 p = P_[a] + (P_[b] - P_[a]) * t;
        int id = (int)nP_.size();
        nP_.push_back(p);
        nok_.push_back(0);
        hits_.push_back({a, b, id});
        return id;
    };
    nfo_.clear(); nfv_.clear(); nfn_.clear();
    nfo_.push_back(0);
    auto close_face = [&](size_t start, int fnb) {
        // drop consecutive duplicates (cyclically)
        size_t w = start;
        for (size_t r = start; r < nfv_.size(); ++r)
            if (w == start || nfv_[w - 1] != nfv_[r]) nfv_[w++] = nfv_[r];
        nfv_.resize(w);
        while (nfv_.size() - start >= 2 && nfv_.back() == nfv_[start]) nfv_.pop_back();
        if (nfv_.size() - start >= 3) {
            nfo_.push_back((int)nfv_.size());
            nfn_.push_back(fnb);
        } else {
            nfv_.resize(start);
        }
    };
    const int nf = (int)fn_.size();
    for (int f = 0; f < nf; ++f) {
        const int b0 = fo_[f], m = fo_[f + 1] - fo_[f];
        size_t start = nfv_.size();
        for (int k = 0; k < m; ++k) {
            const int a = fv_[b0 + k], b = fv_[b0 + (k + 1) % m];
            if (s_[a] <= tol) nfv_.push_back(map_[a]);
            if (s_[a] < -tol && s_[b] > tol) nfv_.push_back(edge_point(a, b));
            else if (s_[a] > tol && s_[b] < -tol) nfv_.push_back(edge_point(b, a));
        }
        close_face(start, fn_[f]);
    }
    // cap polygon: every surviving vertex that lies on the plane
    const int nn = (int)nP_.size();
    ref_.assign(nn, 0);
    for (int x : nfv_) ref_[x] = 1;
    cap_.clear();
    for (int i = 0; i < nv; ++i)
        if (map_[i] >= 0 && s_[i] >= -tol && ref_[map_[i]]) cap_.push_back(map_[i]);
    for (int i = n_kept; i < nn; ++i)
        if (ref_[i]) cap_.push_back(i);
    // merge near-coincident cap vertices (degenerate, e.g. cospherical, configurations)
    const double mt2 = (4.0 * eps_) * (4.0 * eps_);
    mrg_.resize(nn);
    for (int i = 0; i < nn; ++i) mrg_[i] = i;
    bool merged = false;
    for (size_t i = 0; i < cap_.size(); ++i) {
        if (mrg_[cap_[i]] != cap_[i]) continue;
        for (size_t j = i + 1; j < cap_.size(); ++j) {
            if (mrg_[cap_[j]] != cap_[j]) continue;
            if (d2(nP_[cap_[i]], nP_[cap_[j]]) <= mt2) { mrg_[cap_[j]] = cap_[i]; merged = true; }
        }
    }
    if (merged) {
        // rewrite all faces through the merge map
        std::vector<int> ofo(nfo_), ofv(nfv_), ofn(nfn_);
        nfo_.clear(); nfv_.clear(); nfn_.clear();
        nfo_.push_back(0);
        for (size_t f = 0; f + 1 < ofo.size(); ++f) {
            size_t start = nfv_.size();
            for (int k = ofo[f]; k < ofo[f + 1]; ++k) nfv_.push_back(mrg_[ofv[k]]);
            close_face(start, ofn[f]);
        }
        size_t w = 0;
        for (size_t i = 0; i < cap_.size(); ++i)
            if (mrg_[cap_[i]] == cap_[i]) cap_[w++] = cap_[i];
        cap_.resize(w);
    }
    if (cap_.size() >= 3) {
        V3 c{0, 0, 0};
        for (int x : cap_) c = c + nP_[x];
        c = c * (1.0 / (double)cap_.size());
        const V3 un = n * (1.0 / nl);
        V3 ax = std::fabs(un.x) <= std::fabs(un.y) && std::fabs(un.x) <= std::fabs(un.z)
                    ? V3{1, 0, 0}
                    : (std::fabs(un.y) <= std::fabs(un.z) ? V3{0, 1, 0} : V3{0, 0, 1});
        V3 e1 = cross(un, ax);
        e1 = e1 * (1.0 / len(e1));
        const V3 e2 = cross(un, e1);
        std::vector<std::pair<double, int>> ang;
        ang.reserve(cap_.size());
        for (int x : cap_) {
            V3 r = nP_[x] - c;
            ang.push_back({std::atan2(dot(r, e2), dot(r, e1)), x});
        }
        std::sort(ang.begin(), ang.end());
        size_t start = nfv_.size();
        for (auto& a : ang) nfv_.push_back(a.second);
        close_face(start, nb);
    }
    // compact: drop vertices no face references
    ref_.assign(nn, 0);
    for (int x : nfv_) ref_[x] = 1;
    tmp_.assign(nn, -1);
    P_.clear(); ok_.clear();
    for (int i = 0; i < nn; ++i)
        if (ref_[i]) { tmp_[i] = (int)P_.size(); P_.push_back(nP_[i]); ok_.push_back(nok_[i]); }
    fv_.resize(nfv_.size());
    for (size_t k = 0; k < nfv_.size(); ++k) fv_[k] = tmp_[nfv_[k]];
    fo_ = nfo_;
    fn_ = nfn_;
    return true;
}

Box CellClipper::clipped_box(uint32_t site, const Box& b) {
    const V3 v = S_[site];
    const V3 lo = b.lo - v, hi = b.hi - v;
    clip(V3{1, 0, 0}, hi.x, -11);
    clip(V3{-1, 0, 0}, -lo.x, -12);
    clip(V3{0, 1, 0}, hi.y, -13);
    clip(V3{0, -1, 0}, -lo.y, -14);
    clip(V3{0, 0, 1}, hi.z, -15);
    clip(V3{0, 0, -1}, -lo.z, -16);
    Box out;
    for (const V3& p : P_) out.add(v + p);
    return out;
}

void CellClipper::compute(uint32_t site, std::vector<V3>& corners, std::vector<uint32_t>* nbrs) {
    const V3 v = S_[site];
    init_box(v);
    auto is_sentinel = [&](uint32_t w) {
        for (int k = 0; k < nsent_; ++k)
            if (sent_[k] == w) return true;
        return false;
    };
    auto bisect = [&](uint32_t w) {
        const V3 n = S_[w] - v;
        const double nn2 = sq(n);
        if (nn2 == 0.0) return false;
        return clip(n, 0.5 * nn2, (int)w);
    };
    for (int k = 0; k < nsent_; ++k)
        if (sent_[k] != site) bisect(sent_[k]);
    tree_.knn(v, k_, site, knn_);
    for (auto& kv : knn_)
        if (!is_sentinel(kv.second)) bisect(kv.second);
    // certify corners: the owner must be a nearest site of every corner (empty-ball property)
    for (int guard = 0; guard < 1000000; ++guard) {
        bool clipped = false;
        for (size_t i = 0; i < P_.size(); ++i) {
            if (ok_[i]) continue;
            const V3 u = v + P_[i];
            double dw;
            const uint32_t w = tree_.nearest(u, d2(u, v), &dw);
            if (w == UINT32_MAX || w == site) { ok_[i] = 1; continue; }
            const V3 n = S_[w] - v;
            const double nn2 = sq(n);
            if (nn2 > 0.0 && dot(P_[i], n) - 0.5 * nn2 > eps_ * std::sqrt(nn2)) {
                if (clip(n, 0.5 * nn2, (int)w)) { clipped = true; break; }
            }
            ok_[i] = 1;
        }
        if (!clipped) break;
    }
    corners.resize(P_.size());
    for (size_t i = 0; i < P_.size(); ++i) corners[i] = v + P_[i];
    if (nbrs) {
        nbrs->clear();
        for (int x : fn_)
            if (x >= 0) nbrs->push_back((uint32_t)x);
        std::sort(nbrs->begin(), nbrs->end());
        nbrs->erase(std::unique(nbrs->begin(), nbrs->end()), nbrs->end());
    }
}

}  // namespace p2m
