// p2m_tables.cu -- build_all_tables on the GPU (REF/SPEC.md:397-423).
//
// The host builder computes every site's Voronoi cell and the closed balls whose union bounds the
// cell's nearest-face region (Theorem 1); this file runs the ball -> face enumeration
// (REF/SPEC.md:192-200), which is embarrassingly parallel over balls:
//   1. k_ball_walk (count)  -- one thread per ball walks a device copy of the builder's own BVH
//                              (box test box_sqdist(c) <= r2 at every node from the root) and counts
//                              the faces it meets: a vertex within r2, or closest_tri(c, f) <= r2;
//   2. exclusive scan of the counts -> each ball's slot range; sites are split into chunks whose
//      hit count fits the device budget;
//   3. k_ball_walk (write)  -- the same walk writes key = site << 32 | face;
//   4. radix sort + unique of the keys -> per-site ascending, duplicate-free lists.
// The walk evaluates the same fp64 expressions in the same order as bvh.cpp (BallWalk) with no
// contraction (--fmad=false), and a ball reaches a leaf iff every box on the root path passes for
// it -- exactly the host's active-set recursion -- so the tables are bit-identical to p2m_build's.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "../../../include/p2m.h"
#include "p2m_device.cuh"

#define P2M_API extern "C" __attribute__((visibility("default")))

extern "C" void p2m_set_last_error_internal(const char* msg);  // libp2m_host.so

namespace {

using p2m::dev::V;
using p2m::dev::vd2;

constexpr int kStack = 96;

struct Job {
    const double4* ball;   // centre xyz, r2
    const uint32_t* ball_site;
    uint64_t n_balls;
    const double* tri;     // 9 per face
    const double* nbox;    // 6 per node
    const uint4* nmeta;    // right, first, count, 0
    const uint32_t* perm;
};

// squared distance from p to the box, 0 inside: same sum order as Box::sqdist (geom.hpp)
__device__ __forceinline__ double box_sqdist(const double* b, V p) {
    double s = 0.0;
    const double pv[3] = {p.x, p.y, p.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double v = pv[k], l = __ldg(b + k), h = __ldg(b + 3 + k);
        if (v < l) s += (l - v) * (l - v);
        else if (v > h) s += (v - h) * (v - h);
    }
    return s;
}

// WRITE = false: out_count[i] = hits of ball i.  WRITE = true: keys at out_keys[pos[i] - base].
template <bool WRITE>
__global__ void __launch_bounds__(128) k_ball_walk(Job j, uint64_t b0, uint64_t b1, uint64_t* out_count,
                                                   const uint64_t* pos, uint64_t base, uint64_t* out_keys,
                                                   int* overflow) {
    const uint64_t i = b0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= b1) return;
    const double4 bl = j.ball[i];
    const V c{bl.x, bl.y, bl.z};
    const double r2 = bl.w;
    uint64_t w = WRITE ? pos[i] - base : 0;
    const uint64_t key_hi = WRITE ? (uint64_t)j.ball_site[i] << 32 : 0;
    uint32_t cnt = 0;
    uint32_t st[kStack];
    int sp = 0;
    if (box_sqdist(j.nbox, c) <= r2) st[sp++] = 0;
    while (sp) {
        const uint32_t n = st[--sp];
        const uint4 m = __ldg(j.nmeta + n);
        if (m.z) {
            for (uint32_t k = m.y; k < m.y + m.z; ++k) {
                const uint32_t f = __ldg(j.perm + k);
                const double* t = j.tri + 9 * (uint64_t)f;
                const V a{__ldg(t), __ldg(t + 1), __ldg(t + 2)};
                const V b{__ldg(t + 3), __ldg(t + 4), __ldg(t + 5)};
                const V cc{__ldg(t + 6), __ldg(t + 7), __ldg(t + 8)};
                bool hit = vd2(a, c) <= r2 || vd2(b, c) <= r2 || vd2(cc, c) <= r2;
                if (!hit) {
                    V p;
                    hit = p2m::dev::closest_tri(c, a, b, cc, &p) <= r2;
                }
                if (hit) {
                    if (WRITE) out_keys[w++] = key_hi | f;
                    ++cnt;
                }
            }
            continue;
        }
        // children: left = n + 1, right = m.x; push right first so the left subtree is walked first
        const uint32_t kids[2] = {m.x, n + 1};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (box_sqdist(j.nbox + 6 * (uint64_t)kids[q], c) <= r2) {
                if (sp < kStack) st[sp++] = kids[q];
                else atomicExch(overflow, 1);
            }
        }
    }
    if (!WRITE) out_count[i] = cnt;
}

__global__ void k_fill_ball_site(const uint64_t* ball_off, uint64_t n_sites, uint32_t* ball_site) {
    const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (s >= n_sites) return;
    for (uint64_t b = ball_off[s]; b < ball_off[s + 1]; ++b) ball_site[b] = (uint32_t)s;
}

__global__ void k_gather_pos(const uint64_t* pos, const uint64_t* ball_off, uint64_t n_sites, uint64_t* out) {
    const uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (s <= n_sites) out[s] = pos[ball_off[s]];
}

// unique keys -> face ids and per-site counts
__global__ void k_split_keys(const uint64_t* keys, const uint64_t* n_unique, uint32_t* faces, uint32_t* site_cnt) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= *n_unique) return;
    const uint64_t k = keys[i];
    faces[i] = (uint32_t)k;
    atomicAdd(site_cnt + (k >> 32), 1u);
}

struct DevBuf {
    std::vector<void*> ptrs;
    ~DevBuf() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <class T>
    cudaError_t alloc(T** p, size_t n) {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
        if (e == cudaSuccess) ptrs.push_back(q);
        *p = (T*)q;
        return e;
    }
};

#define CKT(x)                                                                                    \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            p2m_set_last_error_internal((std::string("table job: ") + #x + ": " + cudaGetErrorString(e_)).c_str()); \
            return P2M_ERR_CUDA;                                                                  \
        }                                                                                         \
    } while (0)

int bits_for(uint64_t n) {
    int b = 1;
    while (b < 64 && (1ull << b) <= n) ++b;
    return b;
}

int run_job(int dev, const p2m_table_job* job, uint64_t* off, uint32_t** lists_out) {
    const uint64_t S = job->n_sites, NB = job->ball_off[S];
    *lists_out = nullptr;
    if (S >= (1ull << 32) || job->n_faces >= (1ull << 32)) {
        p2m_set_last_error_internal("table job: more than 2^32 sites or faces");
        return P2M_ERR_INVALID;
    }
    CKT(cudaSetDevice(dev));
    cudaStream_t st;
    CKT(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamDestroy(s); } } sg{st};
    DevBuf B;
    double4* d_ball; uint64_t* d_boff; uint32_t* d_bsite; double* d_tri; double* d_nbox; uint4* d_nmeta;
    uint32_t* d_perm; uint64_t* d_cnt; uint64_t* d_pos; uint64_t* d_spos; int* d_over;
    CKT(B.alloc(&d_ball, NB));
    CKT(B.alloc(&d_boff, S + 1));
    CKT(B.alloc(&d_bsite, NB));
    CKT(B.alloc(&d_tri, 9 * job->n_faces));
    CKT(B.alloc(&d_nbox, 6 * job->n_nodes));
    CKT(B.alloc(&d_nmeta, job->n_nodes));
    CKT(B.alloc(&d_perm, job->n_faces));
    CKT(B.alloc(&d_cnt, NB + 1));
    CKT(B.alloc(&d_pos, NB + 1));
    CKT(B.alloc(&d_spos, S + 1));
    CKT(B.alloc(&d_over, 1));
    std::vector<uint4> meta(job->n_nodes);
    for (uint64_t n = 0; n < job->n_nodes; ++n)
        meta[n] = make_uint4(job->node_meta[3 * n], job->node_meta[3 * n + 1], job->node_meta[3 * n + 2], 0);
    CKT(cudaMemcpyAsync(d_ball, job->balls, 32 * NB, cudaMemcpyHostToDevice, st));
    CKT(cudaMemcpyAsync(d_boff, job->ball_off, 8 * (S + 1), cudaMemcpyHostToDevice, st));
    CKT(cudaMemcpyAsync(d_tri, job->tri, 72 * job->n_faces, cudaMemcpyHostToDevice, st));
    CKT(cudaMemcpyAsync(d_nbox, job->node_box, 48 * job->n_nodes, cudaMemcpyHostToDevice, st));
    CKT(cudaMemcpyAsync(d_nmeta, meta.data(), 16 * job->n_nodes, cudaMemcpyHostToDevice, st));
    CKT(cudaMemcpyAsync(d_perm, job->perm, 4 * job->n_faces, cudaMemcpyHostToDevice, st));
    CKT(cudaMemsetAsync(d_over, 0, sizeof(int), st));
    CKT(cudaMemsetAsync(d_cnt, 0, 8 * (NB + 1), st));
    const unsigned sb = (unsigned)((S + 256) / 256);
    k_fill_ball_site<<<sb, 256, 0, st>>>(d_boff, S, d_bsite);
    CKT(cudaGetLastError());
    Job j{d_ball, d_bsite, NB, d_tri, d_nbox, d_nmeta, d_perm};
    if (job->n_nodes && NB) {
        k_ball_walk<false><<<(unsigned)((NB + 127) / 128), 128, 0, st>>>(j, 0, NB, d_cnt, nullptr, 0, nullptr, d_over);
        CKT(cudaGetLastError());
    }
    // ball slot offsets (one trailing zero count gives the total)
    {
        size_t tb = 0;
        CKT(cub::DeviceScan::ExclusiveSum(nullptr, tb, d_cnt, d_pos, (int64_t)(NB + 1), st));
        void* tmp; CKT(B.alloc((char**)&tmp, tb));
        CKT(cub::DeviceScan::ExclusiveSum(tmp, tb, d_cnt, d_pos, (int64_t)(NB + 1), st));
    }
    k_gather_pos<<<(unsigned)((S + 1 + 255) / 256), 256, 0, st>>>(d_pos, d_boff, S, d_spos);
    CKT(cudaGetLastError());
    std::vector<uint64_t> spos(S + 1);
    int over = 0;
    CKT(cudaMemcpyAsync(spos.data(), d_spos, 8 * (S + 1), cudaMemcpyDeviceToHost, st));
    CKT(cudaMemcpyAsync(&over, d_over, sizeof(int), cudaMemcpyDeviceToHost, st));
    CKT(cudaStreamSynchronize(st));
    if (over) {
        p2m_set_last_error_internal("table job: BVH deeper than the device walk stack");
        return P2M_ERR_INTERNAL;
    }
    const uint64_t total = spos[S];
    // chunk budget: keys + sort buffer + unique output (3 x 8 B per hit) within half the free memory
    size_t fr = 0, tot = 0;
    CKT(cudaMemGetInfo(&fr, &tot));
    uint64_t cap = std::max<uint64_t>(1u << 20, (uint64_t)(fr / 2) / 28);
    for (uint64_t s = 0; s < S; ++s) cap = std::max<uint64_t>(cap, spos[s + 1] - spos[s]);
    cap = std::min<uint64_t>(cap, std::max<uint64_t>(total, 1));
    uint64_t *d_k0, *d_k1, *d_nu;
    uint32_t *d_faces, *d_scnt;
    CKT(B.alloc(&d_k0, cap));
    CKT(B.alloc(&d_k1, cap));
    CKT(B.alloc(&d_faces, cap));
    CKT(B.alloc(&d_scnt, S));
    CKT(B.alloc(&d_nu, 1));
    CKT(cudaMemsetAsync(d_scnt, 0, 4 * std::max<uint64_t>(S, 1), st));
    size_t sort_tb = 0, uniq_tb = 0;
    CKT(cub::DeviceRadixSort::SortKeys(nullptr, sort_tb, d_k0, d_k1, (int64_t)cap, 0, 32 + bits_for(S), st));
    CKT(cub::DeviceSelect::Unique(nullptr, uniq_tb, d_k1, d_k0, d_nu, (int64_t)cap, st));
    void* tmp;
    CKT(B.alloc((char**)&tmp, std::max(sort_tb, uniq_tb)));
    std::vector<uint32_t> lists;
    lists.reserve(total / 4 + 16);
    uint64_t s0 = 0;
    std::vector<uint32_t> chunk_faces;
    while (s0 < S) {
        uint64_t s1 = s0;
        while (s1 < S && spos[s1 + 1] - spos[s0] <= cap) ++s1;
        if (s1 == s0) s1 = s0 + 1;  // cap >= every single site's hits
        const uint64_t n = spos[s1] - spos[s0];
        const uint64_t b0 = job->ball_off[s0], b1 = job->ball_off[s1];
        if (n) {
            k_ball_walk<true><<<(unsigned)((b1 - b0 + 127) / 128), 128, 0, st>>>(j, b0, b1, nullptr, d_pos,
                                                                             spos[s0], d_k0, d_over);
            CKT(cudaGetLastError());
            size_t tb = sort_tb;
            CKT(cub::DeviceRadixSort::SortKeys(tmp, tb, d_k0, d_k1, (int64_t)n, 0, 32 + bits_for(S), st));
            tb = uniq_tb;
            CKT(cub::DeviceSelect::Unique(tmp, tb, d_k1, d_k0, d_nu, (int64_t)n, st));
            k_split_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_k0, d_nu, d_faces, d_scnt);
            CKT(cudaGetLastError());
            uint64_t nu = 0;
            CKT(cudaMemcpyAsync(&nu, d_nu, 8, cudaMemcpyDeviceToHost, st));
            CKT(cudaStreamSynchronize(st));
            const size_t at = lists.size();
            lists.resize(at + nu);
            CKT(cudaMemcpyAsync(lists.data() + at, d_faces, 4 * nu, cudaMemcpyDeviceToHost, st));
        }
        s0 = s1;
    }
    std::vector<uint32_t> scnt(S);
    if (S) CKT(cudaMemcpyAsync(scnt.data(), d_scnt, 4 * S, cudaMemcpyDeviceToHost, st));
    CKT(cudaStreamSynchronize(st));
    off[0] = 0;
    for (uint64_t s = 0; s < S; ++s) off[s + 1] = off[s] + scnt[s];
    if (off[S] != lists.size()) {
        p2m_set_last_error_internal("table job: per-site counts disagree with the list size");
        return P2M_ERR_INTERNAL;
    }
    uint32_t* out = (uint32_t*)std::malloc(std::max<size_t>(lists.size(), 1) * 4);
    if (!out) {
        p2m_set_last_error_internal("table job: out of host memory");
        return P2M_ERR_OOM;
    }
    if (!lists.empty()) std::memcpy(out, lists.data(), 4 * lists.size());
    *lists_out = out;
    return P2M_OK;
}

}  // namespace

P2M_API int p2m_table_job_device(void* ctx, const p2m_table_job* job, uint64_t* off, uint32_t** lists) {
    if (!job || !off || !lists) {
        p2m_set_last_error_internal("p2m_table_job_device: null pointer");
        return P2M_ERR_INVALID;
    }
    const int dev = ctx ? *(const int*)ctx : 0;
    try {
        return run_job(dev, job, off, lists);
    } catch (const std::bad_alloc&) {
        p2m_set_last_error_internal("table job: out of host memory");
        return P2M_ERR_OOM;
    }
}

P2M_API int p2m_build_device(const double* vertices, uint64_t n_vertices, const uint32_t* faces, uint64_t n_faces,
                             const p2m_build_config* cfg, int device, p2m_host_engine** out) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
        p2m_set_last_error_internal("p2m_build_device: no CUDA device");
        return P2M_ERR_CUDA;
    }
    if (device < 0 || device >= n) {
        p2m_set_last_error_internal("p2m_build_device: bad device id");
        return P2M_ERR_INVALID;
    }
    int dev = device;
    return p2m_build_with(vertices, n_vertices, faces, n_faces, cfg, p2m_table_job_device, &dev, out);
}
