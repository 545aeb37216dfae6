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
    uint32_t* miss = nullptr;       // grouped scan: rows whose list produced no face within the d_min
    uint32_t* miss_n = nullptr;     // seed (a table that is not a Theorem-1 superset), answered by
                                    // launch_table_miss with the exact BVH fallback and flagged
};

cudaError_t launch_morton(const double* q, uint64_t n, const Params& p, uint32_t* keys, uint32_t* rows,
                          cudaStream_t s);
cudaError_t launch_query(const Params& p, const double* q, const uint32_t* rows, uint64_t n, const Out& o,
                         bool counters, cudaStream_t s);
cudaError_t launch_nearest(const Params& p, const double* q, const uint32_t* rows, uint64_t n, uint32_t* site,
                           cudaStream_t s);

// grouped pipeline: (1) descent per row in Morton order -> site key (fallback rows answered inline,
// keyed n_sites so they sort last); (2) [sort by site]; (3) per-CTA tiles of rows sharing a site scan
// the site's list staged through shared memory.
cudaError_t launch_table_miss(const Params& p, const double* q, const Out& o, cudaStream_t s);
cudaError_t launch_descend(const Params& p, const double* q, const uint32_t* rows, uint64_t n,
                           uint32_t* site_key, const Out& o, bool counters, cudaStream_t s);
size_t tiles_tmp_bytes(uint64_t n);
uint64_t max_tiles(uint64_t n, uint64_t n_sites);
size_t tile_order_tmp_bytes(uint64_t max_t);
cudaError_t launch_tile_order(const Params& p, const uint32_t* key, const uint32_t* tiles, uint32_t* meta,
                              uint64_t max_t, uint32_t* tkey, uint32_t* tkey2, uint32_t* tidx, uint32_t* order,
                              void* tmp, size_t tmp_bytes, cudaStream_t s);
cudaError_t launch_tiles(const Params& p, const uint32_t* key, uint64_t n, uint32_t n_sites, uint32_t* hpos, uint32_t* run_start,
                         uint32_t* flag, uint32_t* tix, uint32_t* tiles, uint32_t* meta, void* tmp, size_t tmp_bytes,
                         cudaStream_t s);
cudaError_t launch_scan_tiles(const Params& p, const double* q, const uint32_t* rows, const uint32_t* key,
                              const uint32_t* tiles, const uint32_t* meta, const uint32_t* order, uint64_t n,
                              const Out& o, bool counters, cudaStream_t s, cudaStream_t side = nullptr,
                              cudaEvent_t fork = nullptr, cudaEvent_t join = nullptr);

}  // namespace dev
}  // namespace p2m
