// voronoi.hpp -- bounded Voronoi cells of the site set and their corners (REF/SPEC.md:232-306).
//
// Equivalent construction (documented in DESIGN.md): instead of a global Bowyer-Watson Delaunay
// tetrahedralisation whose incident-tetra circumcentres are the corners (REF/SPEC.md:265-273), each
// site's cell is built directly as a convex polytope:
//   1. start from a box that contains every sentinel-bounded cell, clip by the bisectors of the
//      8 sentinels (REF/SPEC.md:247-255) and of the k nearest sites;
//   2. certify every corner u: if some site w is strictly closer to u than the owner v (beyond
//      the clipping tolerance), clip by bisector(v, w) and repeat.
// Step 2 terminates with exactly the Voronoi cell (up to tolerance): f(x) = |x-v|^2 - |x-w|^2 is
// affine in x, so if any point of the polytope were closer to w, some corner would be -- the
// same argument as the paper's Theorem 1.  Degenerate (cospherical) inputs need no symbolic
// perturbation: near-coincident corners are merged within the tolerance, and a tolerance error
// only ever enlarges a cell, which keeps the interception tables supersets (REF/SPEC.md:435).
#pragma once

#include <cstdint>
#include <vector>

#include "geom.hpp"
#include "sitetree.hpp"

namespace p2m {

class CellClipper {
   public:
    CellClipper(const std::vector<V3>& sites, const SiteTree& tree, const Box& outer,
                const uint32_t* sentinels, int n_sentinels, double eps, int knn_k)
        : S_(sites), tree_(tree), outer_(outer), sent_(sentinels), nsent_(n_sentinels), eps_(eps),
          k_(knn_k) {}

    // corners (absolute positions) and Delaunay neighbours (sites whose bisector bounds a face)
    void compute(uint32_t site, std::vector<V3>& corners, std::vector<uint32_t>* nbrs);

    // After compute(site): clip the cell to box b (the device's cell-locate grid box) and return
    // the bounding box of what remains -- a tight, conservative box of cell ∩ b.  Destroys the cell.
    Box clipped_box(uint32_t site, const Box& b);

    uint64_t clips() const { return clips_; }

   private:
    const std::vector<V3>& S_;
    const SiteTree& tree_;
    Box outer_;
    const uint32_t* sent_;
    int nsent_;
    double eps_;
    int k_;
    uint64_t clips_ = 0;

    // polytope relative to the owning site
    std::vector<V3> P_;
    std::vector<uint8_t> ok_;
    std::vector<int> fo_, fv_, fn_;  // face offsets (size nf+1), cyclic vertex ids, neighbour
    // scratch
    std::vector<V3> nP_;
    std::vector<uint8_t> nok_;
    std::vector<int> nfo_, nfv_, nfn_, map_, cap_, tmp_, ref_, mrg_;
    std::vector<double> s_;
    std::vector<std::pair<double, uint32_t>> knn_;
    struct EdgeHit { int a, b, id; };
    std::vector<EdgeHit> hits_;

    void init_box(V3 v);
    bool clip(V3 n, double d, int nb);
};

}  // namespace p2m
