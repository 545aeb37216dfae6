// p2m_kernels.cuh -- launch interface of the query kernels (p2m_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "p2m_device.cuh"

namespace p2m {
namespace dev {

struct Out {
    double* dist;
    double* cp;
    uint32_t* face;
    uint32_t* site;
    uint32_t* flags;
    uint64_t* per_query;            // optional: 3 per row (candidates, exact, kd nodes)
    unsigned long long* agg;        // optional: candidates, exact, kd nodes, fallbacks
};

cudaError_t launch_morton(const double* q, uint64_t n, const Params& p, uint32_t* keys, uint32_t* rows,
                          cudaStream_t s);
cudaError_t launch_query(const Params& p, const double* q, const uint32_t* rows, uint64_t n, const Out& o,
                         bool counters, cudaStream_t s);
cudaError_t launch_nearest(const Params& p, const double* q, const uint32_t* rows, uint64_t n, uint32_t* site,
                           cudaStream_t s);

}  // namespace dev
}  // namespace p2m
