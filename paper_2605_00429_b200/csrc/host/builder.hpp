// builder.hpp -- the host build phase (REF/SPEC.md:112-456, cmd_build REF/SPEC.md:598-606).
// Preprocessing is produced once on the host and uploaded; it is reported, not optimised
// (BASELINE.json north_star).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/p2m.h"
#include "bvh.hpp"
#include "geom.hpp"
#include "sitetree.hpp"

namespace p2m {

struct GeometryErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct HostEngine {
    p2m_build_config cfg{};
    p2m_build_stats stats{};
    // validated mesh (REF/SPEC.md:132-140)
    std::vector<double> V;
    std::vector<uint32_t> F;
    std::vector<double> tri;     // 9 per face
    std::vector<double> sphere;  // 4 per face (REF geom.cpp:96-120)
    Bvh bvh;
    Box aabb, D, sentinel_box;
    // site set (REF/SPEC.md:237-240): mesh vertices, then 8 sentinels, then auxiliaries
    std::vector<V3> sites;
    std::vector<double> site_xyz;
    std::vector<uint8_t> kind;
    std::vector<double> refs;    // aux projection (3 per site, NaN otherwise)
    std::vector<double> cell_box;  // AABB of each site's Voronoi cell corners (6 per site, NaN for sentinels)
    uint32_t sentinel_ids[8];
    // interception index (REF/SPEC.md:391-394) as CSR
    std::vector<uint64_t> off;
    std::vector<uint32_t> lists;
    // Delaunay adjacency (facet neighbours of the final cells, symmetrised) as CSR
    std::vector<uint64_t> adj_off;
    std::vector<uint32_t> adj;
    uint64_t mesh_hash = 0;
    // final site tree, kept to recompute cell corners on demand
    SiteTree tree;
    double eps = 0.0;
};

// Throws std::invalid_argument / std::runtime_error with a message; the C ABI maps them.
// table_fn != nullptr: the table phase is delegated (p2m_build_with, include/p2m.h)
std::unique_ptr<HostEngine> build_engine(const double* v, uint64_t nv, const uint32_t* f,
                                         uint64_t nf, const p2m_build_config& cfg,
                                         p2m_table_fn table_fn = nullptr, void* table_ctx = nullptr);
std::unique_ptr<HostEngine> build_engine_mesh_only(const double* v, uint64_t nv, const uint32_t* f,
                                                   uint64_t nf, const p2m_build_config& cfg);
void cell_corners(const HostEngine& h, uint32_t site, std::vector<V3>& out);
uint64_t hash_mesh(const double* v, uint64_t nv, const uint32_t* f, uint64_t nf);
void finish_engine(HostEngine& h);  // derived arrays after load
// Delaunay adjacency of an arbitrary point set (facet neighbours of its sentinel-bounded Voronoi
// cells, symmetric, sentinels dropped): the graph of the DelaunayWalk strategy (REF/SPEC.md:476)
void delaunay_adjacency(const double* xyz, uint64_t n, int n_threads, std::vector<uint64_t>& off,
                        std::vector<uint32_t>& adj);


}  // namespace p2m
