// p2m_kernels.cu -- the query-path kernels for sm_100a.
//
//   k_morton        K1  30-bit Morton key of each query in the key box + identity permutation
//   (CUB radix sort) K2  (key, row) pairs -> spatially coherent processing order
//   k_query         K3+K4+K5 fused: per row (in Morton order) the exact nearest-site descent of the
//                   left-balanced k-d tree (stack-free), then the pruned scan of that site's
//                   interception list with the exact point-triangle test, results scattered straight
//                   back to input order.  Rows whose nearest site is a sentinel or that lie outside D
//                   take the exact BVH fallback (K6) in the same kernel.
//
// Semantics restated (REF = /root/reference):
//   nearest_site   REF/SPEC.md:482-487  lexicographic min of (d^2, site id); a subtree is skipped only
//                  when its squared plane distance is STRICTLY above the best d^2
//   query_distance REF/SPEC.md:488-496  d_min = +inf, strict '<', pruned by the per-face sphere; the
//                  prune test |q-c|^2 > (r + d_min + eps)^2 can never skip a face that ties or beats
//                  d_min, so the result is the lexicographic argmin of (d^2, face id) over the list
//   point-triangle REF/proj/src/geom.cpp:31-70 (p2m_device.cuh)
#include <cuda_runtime.h>

#include "p2m_device.cuh"
#include "p2m_kernels.cuh"
#include "p2m_traverse.cuh"

namespace p2m {
namespace dev {

__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v &= 0x3ff;
    v = (v | (v << 16)) & 0x030000FF;
    v = (v | (v << 8)) & 0x0300F00F;
    v = (v | (v << 4)) & 0x030C30C3;
    v = (v | (v << 2)) & 0x09249249;
    return v;
}

__global__ void __launch_bounds__(256) k_morton(const double* __restrict__ q, uint64_t n, Params p,
                                                uint32_t* __restrict__ keys, uint32_t* __restrict__ rows) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double t = (q[3 * i + k] - p.key_lo[k]) * p.key_scale[k];
        t = fmin(fmax(t, 0.0), 1023.0);
        c[k] = (uint32_t)t;
    }
    keys[i] = spread10(c[0]) << 2 | spread10(c[1]) << 1 | spread10(c[2]);
    rows[i] = (uint32_t)i;
}

template <bool kCounters>
__global__ void __launch_bounds__(256) k_query(Params p, const double* __restrict__ q_xyz,
                                               const uint32_t* __restrict__ rows, uint64_t n, Out o) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t cand = 0, exact = 0, visited = 0, fb = 0;
    if (i < n) {
        const uint32_t row = rows ? rows[i] : (uint32_t)i;
        const V q{q_xyz[3 * (uint64_t)row], q_xyz[3 * (uint64_t)row + 1], q_xyz[3 * (uint64_t)row + 2]};
        const NN nn = nearest_site(p, q);
        visited = nn.visited;
        uint32_t flags = 0;
        const bool in_d = q.x >= p.dmin[0] && q.x <= p.dmax[0] && q.y >= p.dmin[1] && q.y <= p.dmax[1] &&
                          q.z >= p.dmin[2] && q.z <= p.dmax[2];
        if (!in_d) flags |= 2u;
        double best = __longlong_as_double(0x7ff0000000000000ll);
        uint32_t bf = 0xffffffffu;
        if (nn.sentinel || !in_d) {
            flags |= 1u;
            fb = 1;
            bf = bvh_closest(p, q, &best);
        } else {
            const uint64_t beg = p.off[nn.id], end = p.off[nn.id + 1];
            cand = end - beg;
            double dmin = __longlong_as_double(0x7ff0000000000000ll);
            for (uint64_t j = beg; j < end; ++j) {
                const uint32_t f = p.lf[j];
                const D4* rec = p.rec + 4 * (uint64_t)f;
                const D4 sp = ldg4(rec);
                const double dc2 = vd2(q, V{sp.x, sp.y, sp.z});
                const double t = sp.w + dmin + p.prune_eps;
                if (dc2 > t * t) continue;
                V a, b, c, pp;
                load_tri(rec, &a, &b, &c);
                const double dd = closest_tri(q, a, b, c, &pp);
                ++exact;
                if (dd < best) { best = dd; bf = f; dmin = sqrt(dd); }
            }
        }
        V cp{__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll),
             __longlong_as_double(0x7ff8000000000000ll)};
        if (bf != 0xffffffffu) {
            V a, b, c;
            load_tri(p.rec + 4 * (uint64_t)bf, &a, &b, &c);
            closest_tri(q, a, b, c, &cp);
        }
        o.dist[row] = sqrt(best);
        o.cp[3 * (uint64_t)row] = cp.x;
        o.cp[3 * (uint64_t)row + 1] = cp.y;
        o.cp[3 * (uint64_t)row + 2] = cp.z;
        o.face[row] = bf;
        o.site[row] = nn.id;
        if (o.flags) o.flags[row] = flags;
        if (kCounters && o.per_query) {
            o.per_query[3 * (uint64_t)row] = cand;
            o.per_query[3 * (uint64_t)row + 1] = exact;
            o.per_query[3 * (uint64_t)row + 2] = visited;
        }
    }
    if (kCounters && o.agg) {
        unsigned long long v[4] = {cand, exact, visited, fb};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], s);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(o.agg + 0, v[0]);
            atomicAdd(o.agg + 1, v[1]);
            atomicAdd(o.agg + 2, v[2]);
            atomicAdd(o.agg + 3, v[3]);
        }
    }
}

__global__ void __launch_bounds__(256) k_nearest(Params p, const double* __restrict__ q_xyz,
                                                 const uint32_t* __restrict__ rows, uint64_t n,
                                                 uint32_t* __restrict__ site) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t row = rows ? rows[i] : (uint32_t)i;
    const V q{q_xyz[3 * (uint64_t)row], q_xyz[3 * (uint64_t)row + 1], q_xyz[3 * (uint64_t)row + 2]};
    site[row] = nearest_site_any(p, q).id;
}

// ---- launchers ----
cudaError_t launch_morton(const double* q, uint64_t n, const Params& p, uint32_t* keys, uint32_t* rows,
                          cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_morton<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(q, n, p, keys, rows);
    return cudaGetLastError();
}

cudaError_t launch_query(const Params& p, const double* q, const uint32_t* rows, uint64_t n, const Out& o,
                         bool counters, cudaStream_t s) {
    if (!n) return cudaSuccess;
    const unsigned g = (unsigned)((n + 255) / 256);
    if (counters) k_query<true><<<g, 256, 0, s>>>(p, q, rows, n, o);
    else k_query<false><<<g, 256, 0, s>>>(p, q, rows, n, o);
    return cudaGetLastError();
}

cudaError_t launch_nearest(const Params& p, const double* q, const uint32_t* rows, uint64_t n, uint32_t* site,
                           cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_nearest<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, q, rows, n, site);
    return cudaGetLastError();
}

}  // namespace dev
}  // namespace p2m
