// bvh.hpp -- axis-aligned BVH over mesh triangles (REF/SPEC.md:172-230).
// Median split of face centroids on the longest centroid-box axis, leaf size 4
// (REF/SPEC.md:216).  Flattened depth-first: left child = node+1, right child stored.
// Used at build time for (multi-)sphere enumeration (table construction, REF/SPEC.md:192-200)
// and exact closest point (aux-site projection and the fallback, REF/SPEC.md:201-209).
#pragma once

#include <cstdint>
#include <vector>

#include "geom.hpp"

namespace p2m {

struct BvhNode {
    Box box;
    uint32_t right;  // interior: index of right child; leaf: unused
    uint32_t first;  // leaf: first index into perm
    uint32_t count;  // leaf: number of faces (0 = interior)
};

struct Ball {
    V3 c;
    double r2;
};

class Bvh {
   public:
    Bvh() = default;
    void build(const double* tri, uint64_t nf, int leaf_size = 4);

    // exact closest point on the mesh, lowest face id on exact d^2 ties
    uint32_t closest(V3 q, double* d2out, V3* pout) const;

    // all faces f with closest_tri(c_k, f) <= r2_k for some ball k (closed balls), appended to out
    // (unsorted, unique).  mark is a per-thread scratch of size nf (zeroed on return).
    void balls_query(const Ball* balls, int nballs, std::vector<uint32_t>& out,
                     std::vector<uint8_t>& mark) const;

    const std::vector<BvhNode>& nodes() const { return nodes_; }
    const std::vector<uint32_t>& perm() const { return perm_; }
    uint64_t n_faces() const { return nf_; }

   private:
    const double* tri_ = nullptr;
    uint64_t nf_ = 0;
    std::vector<BvhNode> nodes_;
    std::vector<uint32_t> perm_;
    V3 A(uint32_t f) const { return ld3(tri_ + 9 * (uint64_t)f); }
    V3 B(uint32_t f) const { return ld3(tri_ + 9 * (uint64_t)f + 3); }
    V3 C(uint32_t f) const { return ld3(tri_ + 9 * (uint64_t)f + 6); }
};

}  // namespace p2m
