// meshgen.hpp -- synthetic workloads (BASELINE.json configs 1..5).
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

namespace p2m {

struct Mesh {
    std::vector<double> v;    // 3 per vertex
    std::vector<uint32_t> f;  // 3 per face
};

Mesh icosphere(int level);
Mesh mesh_config(int cfg);
void gen_queries(int cfg, const double* v, uint64_t nv, const uint32_t* f, uint64_t nf,
                 uint64_t first, uint64_t count, double* out);
void gen_uniform(uint64_t seed, const double* lo, const double* hi, uint64_t first, uint64_t count,
                 double* out);

}  // namespace p2m
