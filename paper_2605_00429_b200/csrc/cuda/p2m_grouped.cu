// p2m_grouped.cu -- the site-grouped query pipeline (default scan mode).
//
// Why: on the benchmark configs almost all scan work sits in interception lists of thousands of
// faces that hundreds of queries share (the auxiliary sites inside closed surfaces), so scanning
// each list once per tile of queries from shared memory turns an L2-bound gather (32 B sphere per
// query per candidate) into a broadcast-fed fp32/fp64 compute loop.
//
//   k_descend       nearest_site (REF/SPEC.md:482-487) per row in Morton order -> site key; rows
//                   outside D or nearest to a sentinel are answered here by the exact BVH fallback
//                   (REF/SPEC.md:491) and keyed n_sites so the regroup sort moves them to the end
//   (CUB radix sort of (site key, row); stable -> Morton order kept inside a site group)
//   k_scan_grouped  CTA = 256 consecutive rows of the site-sorted order.  For each run of rows that
//                   share a site, the CTA stages the site's list 256 entries at a time (face id,
//                   fp64 sphere, fp32 sphere) in shared memory; every member thread scans the staged
//                   chunk IN LIST ORDER for its own query (query_distance, REF/SPEC.md:488-496), so
//                   its d_min evolves exactly as in the sequential oracle and even the counters match.
//
// Pruning per candidate, two stages, both conservative:
//   fp32: skip iff |q_f - c_f|^2 > ((r_up + dmin_up + delta) * (1 + 1e-6))^2, where delta bounds the
//         fp32 rounding of coordinates (4*sqrt(3)*2^-24*M, M = max |coordinate| of D) plus 2 eps.
//         Whenever it skips, the fp64 test below would also skip.
//   fp64: the oracle's test, |q-c|^2 > (r + d_min + eps)^2, then the exact point-triangle kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "p2m_device.cuh"
#include "p2m_kernels.cuh"
#include "p2m_traverse.cuh"

namespace p2m {
namespace dev {

namespace {

constexpr int kTile = 256;


#ifndef P2M_DESC_MINB
#define P2M_DESC_MINB 5   // 48 registers, 5 CTAs/SM: the descent is load-latency bound (measured 0.77 -> 0.67 ms on c2)
#endif
template <bool kCounters>
__global__ void __launch_bounds__(256, P2M_DESC_MINB) k_descend(Params p, const double* __restrict__ q_xyz,
                                                 const uint32_t* __restrict__ rows, uint64_t n,
                                                 uint32_t* __restrict__ site_key, Out o) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t visited = 0, fb = 0;
    if (i < n) {
        const uint32_t row = rows[i];
        const V q{q_xyz[3 * (uint64_t)row], q_xyz[3 * (uint64_t)row + 1], q_xyz[3 * (uint64_t)row + 2]};
        const NN nn = nearest_site_any(p, q);
        visited = nn.visited;
        const bool in_d = q.x >= p.dmin[0] && q.x <= p.dmax[0] && q.y >= p.dmin[1] && q.y <= p.dmax[1] &&
                          q.z >= p.dmin[2] && q.z <= p.dmax[2];
        uint32_t flags = in_d ? 0u : 2u;
        o.site[row] = nn.id;
        if (nn.sentinel || !in_d) {
            flags |= 1u;
            fb = 1;
            double best;
            const uint32_t bf = bvh_closest(p, q, &best);
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
            site_key[i] = p.n_nodes;  // sorts after every real site
            if (kCounters && o.per_query) {
                o.per_query[3 * (uint64_t)row] = 0;
                o.per_query[3 * (uint64_t)row + 1] = 0;
            }
        } else {
            site_key[i] = nn.id;
        }
        if (o.flags) o.flags[row] = flags;
        if (kCounters && o.per_query) o.per_query[3 * (uint64_t)row + 2] = visited;
    }
    if (kCounters && o.agg) {
        unsigned long long v0 = visited, v1 = fb;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            v0 += __shfl_down_sync(0xffffffffu, v0, s);
            v1 += __shfl_down_sync(0xffffffffu, v1, s);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(o.agg + 2, v0);
            atomicAdd(o.agg + 3, v1);
        }
    }
}

// ---- tile construction over the site-sorted order --------------------------------------------
// tiles = maximal runs of equal site key cut every kTile rows; fallback rows (key == n_sites) are
// excluded.  hpos[i] = i at a run head else 0 -> inclusive max-scan gives each row its run start.
__global__ void __launch_bounds__(256) k_run_heads(const uint32_t* __restrict__ key, uint64_t n,
                                                   uint32_t* __restrict__ hpos) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    hpos[i] = (i == 0 || key[i] != key[i - 1]) ? (uint32_t)i : 0u;
}

// Tile height: kTile rows, or p.long_tile rows for "heavy" sites (many exact evaluations expected
// per query, p.heavy, estimated at engine creation), so replicas split their lists and a heavy
// site spreads over more SMs.
__global__ void __launch_bounds__(256) k_tile_flags(Params p, const uint32_t* __restrict__ key,
                                                    const uint32_t* __restrict__ run_start, uint64_t n,
                                                    uint32_t n_sites, uint32_t* __restrict__ flag,
                                                    uint32_t* __restrict__ meta) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = key[i];
    const uint32_t rs = run_start[i];
    uint32_t T = kTile;
    if (k < n_sites) {
        if (p.heavy[k]) T = p.long_tile;
        else if (p.warp_min_chunks && p.coff[k + 1] - p.coff[k] >= p.warp_min_chunks) T = 32;  // warp tiles
    }
    if (p.warp_tiles) T = 32;
    flag[i] = (k < n_sites && ((uint32_t)i == rs || (((uint32_t)i - rs) % T) == 0)) ? 1u : 0u;
    // number of table rows (fallback rows sort last)
    const bool last_valid = k < n_sites && (i + 1 == n || key[i + 1] >= n_sites);
    if (last_valid) meta[1] = (uint32_t)(i + 1);
    if (i == 0 && k >= n_sites) meta[1] = 0;
    if (i == 0) { meta[2] = 0; meta[3] = 0; }  // small tiles (k_tile_keys), table misses (scan)
}

__global__ void __launch_bounds__(256) k_tile_write(const uint32_t* __restrict__ flag,
                                                    const uint32_t* __restrict__ tix, uint64_t n,
                                                    uint32_t* __restrict__ tiles, uint32_t* __restrict__ meta) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (flag[i]) tiles[tix[i]] = (uint32_t)i;
    if (i + 1 == n) meta[0] = tix[i] + flag[i];
}

// ---- the tile scan --------------------------------------------------------------------------
// packed fp32 pairs (sm_100a f32x2): two candidates per instruction in the pre-filter
__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t add2_up(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rp.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t mul2_up(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rp.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ uint64_t add2_dn(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t sub2_up(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rp.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t mul2_dn(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fma2_dn(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// ---- bounding-cylinder lower bound ------------------------------------------
// A record {c, 4R^2}, {n, t} (p2m_engine.cu fit_cyl) encloses every member face: |nn.(x-c)| <= t and
// in-plane distance <= R (nn = n/|n|).  For the fp32 query q_f, v = q_f - c, h = n.v, S = |v|^2:
//   d(q_f, cylinder)^2 = a^2 + max(0, rho - R)^2,  a = max(0, |h| - t),  rho^2 = S - h^2.
// The stored t already covers the fp32 error of |h| (40 * 2^-24 * M, M = max |coordinate| of D), and
// rho^2 is lowered by kRhoErr * S, which covers the rounding of S and h^2; every later step rounds
// toward the safe side, so "pruned" below implies d(q_f, cylinder) > U.  U is the row's d_min bound
// (DK: rounded up, plus the fp32 rounding slack of q, times 1 + 1e-6), so a pruned face can neither
// beat nor tie the row's (d^2, face id) minimum.  Square-free: with rho_lo > R,
//   (rho - R)^2 + a^2 > U^2  <=>  B > 2 R rho,  B = rho^2 + R^2 + a^2 - U^2  <=>  B > 0 && B^2 > 4R^2 rho^2.
// For one face (t ~ 0, R = its min-enclosing radius) this is the distance to its bounding disk: on
// c5, 5 faces per query pass it against 334 for the bounding sphere (same final d_min).
constexpr float kRhoErr = 24.0f / 16777216.0f;   // 24 * 2^-24
// Per-row fp32 error scale Mq = max(|q_f|_inf, mesh_m) (every centre, point and mesh coordinate is
// within mesh_m): |q - q_f| <= sqrt(3) u Mq, an fp32 point P of the mesh is within sqrt(3) u Mq of
// the exact one, and the cylinder test's |h| is within 21 u Mq of exact.
constexpr float kUbSlack = 6.929e-7f;   // >= 2 * 2 sqrt(3) * 2^-24: rounding of q and of P in |q_f - P_f|
constexpr float kDkSlack = 2.8e-6f;     // >= (4 sqrt(3) + 40) * 2^-24: q rounding in the prunes + |h| error
__device__ __forceinline__ float row_scale(const Params& p, float qx, float qy, float qz) {
    return fmaxf(fmaxf(fabsf(qx), fabsf(qy)), fmaxf(fabsf(qz), p.mesh_m));
}
// the row's pruning bound DK from a rigorous upper bound ub of its distance to the mesh:
// (ub + slack(Mq) + 2 eps) * (1 + 1e-6), rounded up
__device__ __forceinline__ float dk_of(const Params& p, float ub, float Mq) {
    return __fmul_ru(__fadd_ru(ub, __fmaf_ru(Mq, kDkSlack, p.eps2)), 1.000001f);
}
// upper bound of |q - P| from the fp32 d2f = |q_f - P_f|^2 (P on the mesh)
__device__ __forceinline__ float ub_of(float d2f, float Mq) {
    return __fadd_ru(__fmul_ru(__fsqrt_ru(d2f), 1.000001f), __fmul_ru(Mq, kUbSlack));
}

// may some point of the cylinder lie within U of q_f (U2 = U^2 rounded up)?  false = prune
__device__ __forceinline__ bool cyl_near(float qx, float qy, float qz, float U2, float4 c0, float4 c1) {
    const float vx = qx - c0.x, vy = qy - c0.y, vz = qz - c0.z;
    const float h = __fmaf_rn(vz, c1.z, __fmaf_rn(vy, c1.y, __fmul_rn(vx, c1.x)));
    const float S = __fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx)));
    const float rl = __fmaf_rn(S, -kRhoErr, __fmaf_rn(-h, h, S));   // <= rho^2
    const float a = fmaxf(fabsf(h) - c1.w, 0.f);
    const float A = __fmul_rd(a, a);
    if (A > U2) return false;
    if (4.f * rl > c0.w) {                                         // rho_lo > R
        const float nB = __fsub_ru(U2, __fadd_rd(__fmaf_rd(c0.w, 0.25f, rl), A));   // >= -B
        if (nB < 0.f && __fmul_rd(nB, nB) > __fmul_ru(c0.w, rl)) return false;
    }
    return true;
}

// visiting-order key: an (approximate) lower bound of d(q, cylinder)^2 as an ordered uint
__device__ __forceinline__ uint32_t cyl_key(float qx, float qy, float qz, float4 c0, float4 c1) {
    const float vx = qx - c0.x, vy = qy - c0.y, vz = qz - c0.z;
    const float h = __fmaf_rn(vz, c1.z, __fmaf_rn(vy, c1.y, __fmul_rn(vx, c1.x)));
    const float S = __fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx)));
    const float a = fmaxf(fabsf(h) - c1.w, 0.f);
    const float e = fmaxf(__fsqrt_rn(fmaxf(__fmaf_rn(-h, h, S), 0.f)) - 0.5f * __fsqrt_rn(c0.w), 0.f);
    return __float_as_uint(__fmaf_rn(a, a, e * e));
}

// One CTA per tile (all rows share one site).  A tile of m rows uses G = ceil(m/32) warps per
// replica and R = 8 / G replicas; replica r scans the 32-candidate batches b == r (mod R) of every
// staged chunk, so small groups still keep all 8 warps busy.  Per batch, each lane computes a
// pass/prune bit per candidate with the conservative fp32 disk test (branch-free, f32x2), then the
// warp walks the union of set bits in list order: a lane whose bit is set re-tests the disk with its
// CURRENT d_min and, on pass, runs the exact point-triangle kernel on the face record (all lanes read
// the same record: broadcast).  Every prune is conservative, so each row's
// result is the full-list argmin.  Replicas are merged by the lexicographic min of (d^2, face id),
// the sequential argmin.
constexpr int kChunk = 256;
constexpr int kWinChunks = 256;                  // level-0 need bits are computed per window of chunks
static_assert(kWinChunks <= kTile, "one thread per window chunk when ordering");

constexpr int kWarps = kTile / 32;

// Staged disks of one 32-entry batch, pair-interleaved so that every 16-byte load yields two f32x2
// operands: pair pp = candidates (2pp, 2pp+1) occupies 16 floats
//   (cx0,cx1,cy0,cy1) (cz0,cz1,R4_0,R4_1) (nx0,nx1,ny0,ny1) (nz0,nz1,t0,t1)
// stage_disk writes candidate k's record (r0 = {c, 4R^2}, r1 = {n, t}) into that layout.
#define kPadDisk make_float4(1e18f, 1e18f, 1e18f, 0.f)  // record of a padding entry: far away, never passes
__device__ __forceinline__ void stage_disk(float* pf, int k, float4 r0, float4 r1) {
    float* b = pf + 16 * (k >> 1) + (k & 1);
    b[0] = r0.x; b[2] = r0.y; b[4] = r0.z; b[6] = r0.w;
    b[8] = r1.x; b[10] = r1.y; b[12] = r1.z; b[14] = r1.w;
}
__device__ __forceinline__ void staged_disk(const float* pf, int k, float4& r0, float4& r1) {
    const float* b = pf + 16 * (k >> 1) + (k & 1);
    r0 = make_float4(b[0], b[2], b[4], b[6]);
    r1 = make_float4(b[8], b[10], b[12], b[14]);
}

// Level 2 of one staged batch for this lane's row: bit k of the result = candidate k's bounding disk may
// hold a point within the row's d_min bound DK (conservative, branch-free f32x2).  Also tightens DK by
// the nearest staged disk centre (a point of its face up to ctr_slack: an upper bound of the distance).
__device__ __forceinline__ uint32_t batch_mask_row(const Params& p, bool active, uint64_t QX, uint64_t QY, uint64_t QZ,
                                                   uint64_t& DK, const float4* disk, int valid, float* sdk) {
    const float qxf = __uint_as_float((uint32_t)QX), qyf = __uint_as_float((uint32_t)QY), qzf = __uint_as_float((uint32_t)QZ);
    const float Mq = row_scale(p, qxf, qyf, qzf);
    uint32_t mask = 0;
    if (active && sdk) {                         // the row's bound as tightened by the other replicas
        float dkx, dky;
        upk2(DK, dkx, dky);
        const float v = *sdk;
        if (v < dkx) DK = pk2(v, v);
    }
    if (active) {
        float dkx, dky;
        upk2(DK, dkx, dky);
        const float u2 = __fmul_ru(dkx, dkx);
        const uint64_t U2 = pk2(u2, u2);
        const uint64_t NRHO = pk2(-kRhoErr, -kRhoErr), M4 = pk2(-4.f, -4.f), Q = pk2(0.25f, 0.25f);
        float smin = __int_as_float(0x7f800000);  // min |q_f - c|^2 over the batch's disk centres
#pragma unroll 4
        for (int pp = 0; pp < 16; ++pp) {
            const float4 A0 = disk[4 * pp], A1 = disk[4 * pp + 1], A2 = disk[4 * pp + 2], A3 = disk[4 * pp + 3];
            const uint64_t vx = sub2(QX, pk2(A0.x, A0.y));
            const uint64_t vy = sub2(QY, pk2(A0.z, A0.w));
            const uint64_t vz = sub2(QZ, pk2(A1.x, A1.y));
            const uint64_t h = fma2(vz, pk2(A3.x, A3.y), fma2(vy, pk2(A2.z, A2.w), mul2(vx, pk2(A2.x, A2.y))));
            const uint64_t S = fma2(vz, vz, fma2(vy, vy, mul2(vx, vx)));
            const uint64_t rl = fma2(S, NRHO, sub2(S, mul2(h, h)));        // <= rho^2
            {
                float s0, s1;
                upk2(S, s0, s1);
                smin = fminf(smin, fminf(s0, s1));
            }
            float h0, h1;
            upk2(h, h0, h1);
            const float a0 = fmaxf(fabsf(h0) - A3.z, 0.f), a1 = fmaxf(fabsf(h1) - A3.w, 0.f);
            const uint64_t a = pk2(a0, a1);
            const uint64_t AA = mul2_dn(a, a);
            const uint64_t R4 = pk2(A1.z, A1.w);
            const uint64_t n1 = sub2(U2, AA);                             // < 0 iff a^2 > U^2
            const uint64_t n2 = fma2(rl, M4, R4);                         // < 0 iff rho_lo > R
            const uint64_t nB = sub2_up(U2, add2_dn(fma2_dn(R4, Q, rl), AA));   // < 0 => B > 0
            const uint64_t n4 = sub2(mul2_up(R4, rl), mul2_dn(nB, nB));   // < 0 iff B^2 > 4 R^2 rho^2
            float x1a, x1b, x2a, x2b, xBa, xBb, x4a, x4b;
            upk2(n1, x1a, x1b);
            upk2(n2, x2a, x2b);
            upk2(nB, xBa, xBb);
            upk2(n4, x4a, x4b);
            // prune bit = sign(n1) | (sign(n2) & sign(nB) & sign(n4)) (IEEE: an exact zero difference
            // is +0 and never prunes; NaN from inf - inf has its sign bit clear)
            const uint32_t pa = __float_as_uint(x1a) | (__float_as_uint(x2a) & __float_as_uint(xBa) & __float_as_uint(x4a));
            const uint32_t pb = __float_as_uint(x1b) | (__float_as_uint(x2b) & __float_as_uint(xBb) & __float_as_uint(x4b));
            mask = __funnelshift_l(pa, mask, 1);
            mask = __funnelshift_l(pb, mask, 1);
        }
        mask = ~__brev(mask);  // bit k = candidate k passes
        if (valid < 32) mask &= (1u << valid) - 1u;
        // every disk centre is a point of its face (up to ctr_slack): |q - c| bounds the row's distance
        // from above, so the nearest staged centre tightens d_min before the exact tests (padding
        // entries sit at 1e18, kPadDisk, and never count)
        if (p.no_seed != 1) {
            const float dkf = dk_of(p, __fadd_ru(ub_of(smin, Mq), p.ctr_slack), Mq);
            if (dkf < dkx) {
                DK = pk2(dkf, dkf);
                if (sdk) atomicMin(reinterpret_cast<int*>(sdk), __float_as_int(dkf));
            }
        }
    }
    return mask;
}

// One 32-entry batch staged in shared memory (disks: 16 pairs x 64 bytes, fid: 32 face ids), scanned
// for this lane's row.  Called by every lane of the warp.
template <bool kCounters>
__device__ __forceinline__ void scan_batch_row(const Params& p, bool active, const V& q, uint64_t QX, uint64_t QY,
                                               uint64_t QZ, uint64_t& DK, double& best, uint32_t& bf,
                                               uint32_t& exact, unsigned long long& passes,
                                               unsigned long long& rare_iters, unsigned long long& sbytes,
                                               const float4* disk, const uint32_t* fid, int valid, int lane,
                                               float* sdk) {
    const float qxf = __uint_as_float((uint32_t)QX), qyf = __uint_as_float((uint32_t)QY), qzf = __uint_as_float((uint32_t)QZ);
    const float Mq = row_scale(p, qxf, qyf, qzf);
    const uint32_t mask = batch_mask_row(p, active, QX, QY, QZ, DK, disk, valid, sdk);
    uint32_t um = __reduce_or_sync(0xffffffffu, mask);
    if (kCounters) {
        passes += __popc(mask);
        if (lane == 0) rare_iters += 32u * __popc(um);
    }
    // the exact test of one candidate kk of this lane: the disk again with the CURRENT d_min (the batch
    // mask used the d_min of the batch start), then fp64
    auto visit = [&](int kk) -> bool {
        {
            float dkx, dky;
            upk2(DK, dkx, dky);
            float4 r0, r1;
            staged_disk(reinterpret_cast<const float*>(disk), kk, r0, r1);
            if (!cyl_near(qxf, qyf, qzf, __fmul_ru(dkx, dkx), r0, r1)) return false;
        }
        const uint32_t f = fid[kk];
        if (f == bf) return false;               // the deep seed's face: already evaluated
        V a, bb3, c3, pp3;
        load_tri(p.rec + 4 * (uint64_t)f, &a, &bb3, &c3);
        const double dd = closest_tri(q, a, bb3, c3, &pp3);
        ++exact;
        if (dd < best || (dd == best && f < bf)) {
            best = dd;
            bf = f;
            // any upper bound of sqrt(best) is a valid d_min for the prunes: the fp32 sqrt rounded up of
            // best rounded up (cheaper than the fp64 sqrt)
            const float dkf = dk_of(p, __fsqrt_ru(__double2float_ru(dd)), Mq);
            float dkx, dky;
            upk2(DK, dkx, dky);
            if (dkf < dkx) {
                DK = pk2(dkf, dkf);
                if (sdk) atomicMin(reinterpret_cast<int*>(sdk), __float_as_int(dkf));  // >= 0: int order
            }
        }
        return true;
    };
    // the warp walks the union of set bits in list order (the face record read is a broadcast)
    while (um) {
        const int kk = __ffs(um) - 1;
        um &= um - 1;
        bool ex = false;
        if ((mask >> kk) & 1u) ex = visit(kk);
        if (kCounters && __any_sync(0xffffffffu, ex) && lane == 0) sbytes += 96;  // one face record per warp visit
    }
}

// d_min seeds of one row of site s (both are upper bounds of the distance to the mesh, so the
// (d^2, face id) argmin and every face that could tie it survive every prune).
template <bool kCounters>
__device__ __forceinline__ void seed_row(const Params& p, uint32_t s, const V& q, uint64_t QX, uint64_t QY,
                                         uint64_t QZ, double& dmin, uint64_t& DK, double& best, uint32_t& bf,
                                         uint32_t& exact) {
    const float finf = __int_as_float(0x7f800000);
    const float qxf = __uint_as_float((uint32_t)QX), qyf = __uint_as_float((uint32_t)QY), qzf = __uint_as_float((uint32_t)QZ);
    const float Mq = row_scale(p, qxf, qyf, qzf);
    const uint64_t bo = p.boff[s], co = p.coff[s];
    const uint32_t nch = (uint32_t)(p.coff[s + 1] - co);
    if (p.no_seed != 1) {
        // Seed d_min with an upper bound of the distance to the mesh: |q - ref| for a point ref ON
        // the mesh (the site itself for a mesh vertex, proj(s, M) for an auxiliary site).  A face
        // whose lower bound exceeds it (plus the prune slack) cannot attain or tie the minimum, so
        // the (d^2, face) argmin is unchanged; only exact evaluations are saved.  The sequential
        // fused path keeps d_min = +inf (REF/SPEC.md:514) so its counters stay oracle-identical.
        const D4 rf = ldg4(p.site_ref + s);
        if (rf.w != 0.0) {
            dmin = sqrt(vd2(q, V{rf.x, rf.y, rf.z}));
            const float dkf = dk_of(p, __double2float_ru(dmin), Mq);
            DK = pk2(dkf, dkf);
        }
    }
    if (p.no_seed != 1 && !p.no_batch) {
        // Tighter seed: every chunk and batch carries a point P on the mesh near its centre
        // (p2m_engine.cu group_point), so |q - P| bounds the distance to the mesh from above.  fp32
        // with upward rounding: sqrt(d2f)*(1+1e-6) covers the rounding of d2f, delta the fp32
        // rounding of q and of P.  The min runs over every chunk point, then over the batch points
        // of this lane's best chunk.
        float ub = finf;
        uint32_t bc = 0;
        for (uint32_t c2 = 0; c2 < nch; ++c2) {
            const float4 c = p.cpt[co + c2];  // same address across the tile's lanes: broadcast
            const float dx = qxf - c.x, dy = qyf - c.y, dz = qzf - c.z;
            const float d2f = __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz)));
            const float u = ub_of(d2f, Mq);
            if (u < ub) { ub = u; bc = c2; }
        }
        const uint64_t nbl = p.boff[s + 1] - bo;
        const uint64_t bb0 = (uint64_t)bc * (kChunk / 32), bb1 = min(nbl, bb0 + kChunk / 32);
        float ubb = finf;
        uint64_t bbest = bb0;
        for (uint64_t b2 = bb0; b2 < bb1; ++b2) {
            const float4 c = p.bpt[bo + b2];
            const float dx = qxf - c.x, dy = qyf - c.y, dz = qzf - c.z;
            const float d2f = __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz)));
            const float u = ub_of(d2f, Mq);
            if (u < ubb) { ubb = u; bbest = b2; }
        }
        ub = fminf(ub, ubb);
        if ((double)ub < dmin) {
            dmin = (double)ub;
            const float dkf = dk_of(p, ub, Mq);
            DK = pk2(dkf, dkf);
        }
        if (p.no_seed == 0 && nbl) {
            // Deep seed: the face of the row's best batch whose disk centre is nearest to q, evaluated
            // exactly.  It is a face of this list, so (best, bf) starts at a genuine candidate of the
            // argmin and d_min at its exact distance -- within the list's own tolerance of the final
            // answer for most rows, so the chunk, batch and disk tests that follow prune against a
            // near-final bound from the start, whatever order the tile visits the batches in (the
            // best-first order serves the tile's first row only).  All 32 lanes evaluate at once.
            const uint64_t e0 = p.off[s] + 32ull * bbest;
            const int ne = (int)min((uint64_t)32, p.off[s + 1] - e0);
            float sm = finf;
            uint32_t fm = 0;
#pragma unroll 4
            for (int k = 0; k < ne; ++k) {
                const uint32_t f = p.lfs[e0 + k];
                const float4 c = p.fcy[kCy * (uint64_t)f];
                const float dx = qxf - c.x, dy = qyf - c.y, dz = qzf - c.z;
                const float d2f = __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz)));
                if (d2f < sm) { sm = d2f; fm = f; }
            }
            V a, b3, c3, pp3;
            load_tri(p.rec + 4 * (uint64_t)fm, &a, &b3, &c3);
            best = closest_tri(q, a, b3, c3, &pp3);
            bf = fm;
            ++exact;
            const float dkf = dk_of(p, __fsqrt_ru(__double2float_ru(best)), Mq);
            float dkx, dky;
            upk2(DK, dkx, dky);
            if (dkf < dkx) DK = pk2(dkf, dkf);
        }
    }
}

// A deep-seeded row always holds a face, so "the list had no face within |q - ref(site)|" (a table that
// is not a Theorem-1 superset, P2M_FLAG_TABLE_MISS) is detected from the result: ref lies ON the mesh,
// so a superset list's minimum cannot exceed |q - ref| beyond rounding.
__device__ __forceinline__ bool table_miss(const Params& p, uint32_t s, const V& q, double best, uint32_t bf) {
    if (bf == 0xffffffffu) return true;
    if (p.no_seed != 0) return false;
    const D4 rf = ldg4(p.site_ref + s);
    if (rf.w == 0.0) return false;
    const double dr = vd2(q, V{rf.x, rf.y, rf.z});
    return best > dr * (1.0 + 1e-9) + p.prune_eps * p.prune_eps;
}

// ---- warp tiles: one warp per tile of <= 32 rows --------------------------------------------
// A tile of at most 32 rows is scanned by ONE warp (lanes = rows), 8 independent tiles per CTA, with
// no block barrier: the warp walks its site's list on its own.  Chunks are taken in windows of 32
// (lane k holds chunk k's cylinder): a level-0 vote keeps the chunks some row may need, ranked by
// the lower bound of the tile's first row (best-first); each kept chunk is re-tested with the current
// d_min, its batch cylinders are voted on (level 1) in the same best-first order, and each needed
// batch is staged in the warp's shared-memory slice and scanned (level 2 + exact, scan_batch_row).
// Used for the small tiles beside k_scan_tiles (side stream), and for every tile in warp mode
// (Params::warp_tiles: 32-row tiles everywhere, k_scan_tiles not launched).
#ifndef P2M_SMALL_MINB
#define P2M_SMALL_MINB 4
#endif
template <bool kCounters>
__global__ void __launch_bounds__(256, P2M_SMALL_MINB) k_scan_small(Params p, const double* __restrict__ q_xyz,
                                                        const uint32_t* __restrict__ rows,
                                                        const uint32_t* __restrict__ key,
                                                        const uint32_t* __restrict__ tiles,
                                                        const uint32_t* __restrict__ meta,
                                                        const uint32_t* __restrict__ order, Out o) {
    __shared__ float4 s_disk[kWarps][64];
    __shared__ uint32_t s_fid[kWarps][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t nt = meta[0], ns = meta[2];
    const uint32_t ti = blockIdx.x * kWarps + w;
    if (ti >= ns) return;                        // warp-uniform: no block barrier in this kernel
    float4* wd = s_disk[w];
    uint32_t* wf = s_fid[w];
    const uint32_t b = order[nt - ns + ti];
    const uint32_t start = tiles[b];
    const uint32_t stop = (b + 1 < nt) ? tiles[b + 1] : meta[1];
    const int m = (int)(stop - start);
    const uint32_t s = key[start];
    const bool active = lane < m;
    const long long t_start = p.tile_trace ? clock64() : 0;
    const float finf = __int_as_float(0x7f800000);
    uint32_t row = 0;
    V q{0, 0, 0};
    float fx = 0.f, fy = 0.f, fz = 0.f;
    if (active) {
        row = rows[start + lane];
        q = V{q_xyz[3 * (uint64_t)row], q_xyz[3 * (uint64_t)row + 1], q_xyz[3 * (uint64_t)row + 2]};
        fx = (float)q.x; fy = (float)q.y; fz = (float)q.z;
    }
    const uint64_t QX = pk2(fx, fx), QY = pk2(fy, fy), QZ = pk2(fz, fz);
    const float rx = __shfl_sync(0xffffffffu, fx, 0), ry = __shfl_sync(0xffffffffu, fy, 0),
                rz = __shfl_sync(0xffffffffu, fz, 0);  // the tile's first row: visiting order
    double best = __longlong_as_double(0x7ff0000000000000ll), dmin = best;
    uint64_t DK = pk2(finf, finf);
    uint32_t bf = 0xffffffffu, exact = 0;
    unsigned long long passes = 0, rare_iters = 0;
    unsigned long long sbytes = 0;               // structure bytes loaded (counters mode; bench roofline)
    if (active) seed_row<kCounters>(p, s, q, QX, QY, QZ, dmin, DK, best, bf, exact);
    const uint64_t beg = p.off[s], end = p.off[s + 1];
    const uint64_t bo = p.boff[s], co = p.coff[s];
    const uint32_t nch = (uint32_t)(p.coff[s + 1] - co);
    if (kCounters && lane == 0) sbytes += 16ull * nch + 76;  // chunk points, site ref, offsets, tile meta
    // conservative "may some member be within d_min" test of this lane's row against a group cylinder
    auto near = [&](float4 c0, float4 c1) {
        float dkx, dky;
        upk2(DK, dkx, dky);
        return cyl_near(fx, fy, fz, __fmul_ru(dkx, dkx), c0, c1);
    };
    auto bcast = [&](float4 v, int src) {
        return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                           __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
    };
    // best-first order without sorting: take the lane holding the smallest key (ties: the lowest
    // lane) and retire it; keys of the items to visit are < ~0 (non-negative float bits)
    auto take_min = [&](uint32_t& k) {
        const uint32_t mk = __reduce_min_sync(0xffffffffu, k);
        const int src = __ffs(__ballot_sync(0xffffffffu, k == mk)) - 1;
        if (lane == src) k = 0xffffffffu;
        return src;
    };
    float* wdf = reinterpret_cast<float*>(wd);
    for (uint32_t w0 = 0; w0 < nch; w0 += 32) {
        const int wn = (int)min(32u, nch - w0);
        float4 cc0 = make_float4(0.f, 0.f, 0.f, 0.f), cc1 = cc0;  // lane k: chunk w0 + k's cylinder
        if (lane < wn) { cc0 = p.ccy[kCy * (co + w0 + lane)]; cc1 = p.ccy[kCy * (co + w0 + lane) + 1]; }
        if (kCounters && lane == 0) sbytes += 32ull * wn;
        // level 0: the chunks of the window some row may need
        uint32_t cneed = 0;
        if (nch == 1 || p.no_batch) {
            cneed = wn == 32 ? 0xffffffffu : ((1u << wn) - 1u);
        } else {
            for (int k = 0; k < wn; ++k) {
                const float4 c0 = bcast(cc0, k), c1 = bcast(cc1, k);
                if (__any_sync(0xffffffffu, active && near(c0, c1))) cneed |= 1u << k;
            }
        }
        const int nn = __popc(cneed);
        uint32_t ckey = ((cneed >> lane) & 1u) ? (nn > 1 ? cyl_key(rx, ry, rz, cc0, cc1) : 0u) : 0xffffffffu;
        for (int pos = 0; pos < nn; ++pos) {
            const int src = take_min(ckey);
            const uint32_t cidx = w0 + (uint32_t)src;
            if (pos > 0 && !p.no_batch) {        // re-test with the d_min the earlier chunks produced
                const float4 c0 = bcast(cc0, src), c1 = bcast(cc1, src);
                if (!__any_sync(0xffffffffu, active && near(c0, c1))) continue;
            }
            const uint64_t cb = beg + (uint64_t)cidx * kChunk;
            const int nb = (int)((min((uint64_t)kChunk, end - cb) + 31) >> 5);
            if (kCounters && lane == 0) sbytes += 32ull * nb;  // the chunk's batch cylinders
            // the chunk's batches best-first for the first row
            float4 b0c = make_float4(0.f, 0.f, 0.f, 0.f), b1c = b0c;
            uint32_t bk = 0xffffffffu;
            if (lane < nb) {
                const uint64_t gi = kCy * (bo + (uint64_t)cidx * (kChunk / 32) + lane);
                b0c = p.bcy[gi];
                b1c = p.bcy[gi + 1];
                bk = nb > 1 ? cyl_key(rx, ry, rz, b0c, b1c) : 0u;
            }
            for (int bpos = 0; bpos < nb; ++bpos) {
                const int bsrc = take_min(bk);
                if (!p.no_batch) {
                    const float4 c0 = bcast(b0c, bsrc), c1 = bcast(b1c, bsrc);
                    if (!__any_sync(0xffffffffu, active && near(c0, c1))) continue;  // pruned whole
                }
                const uint64_t b0 = cb + 32ull * bsrc;
                const int valid = (int)min((uint64_t)32, end - b0);
                uint32_t f = 0;
                float4 r0 = kPadDisk, r1 = make_float4(0.f, 0.f, 0.f, 0.f);
                if (lane < valid) { f = p.lfs[b0 + lane]; r0 = p.fcy[kCy * (uint64_t)f]; r1 = p.fcy[kCy * (uint64_t)f + 1]; }
                wf[lane] = f;
                stage_disk(wdf, lane, r0, r1);
                __syncwarp();
                if (kCounters && lane == 0) sbytes += 36ull * valid;  // staged ids + disks
                scan_batch_row<kCounters>(p, active, q, QX, QY, QZ, DK, best, bf, exact, passes, rare_iters, sbytes,
                                          wd, wf, valid, lane, nullptr);
                __syncwarp();                    // the slice is rewritten by the next batch
            }
        }
    }
    if (p.tile_trace && lane == 0) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* t = p.tile_trace + 4 * (uint64_t)b;
        t[0] = s; t[1] = (unsigned long long)m; t[2] = end - beg;
        t[3] = (unsigned long long)(clock64() - t_start) << 8 | (smid & 0xff);
    }
    if (active) {
        V cp{__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll),
             __longlong_as_double(0x7ff8000000000000ll)};
        if (bf != 0xffffffffu) {
            V a, bb, c;
            load_tri(p.rec + 4 * (uint64_t)bf, &a, &bb, &c);
            closest_tri(q, a, bb, c, &cp);
        }
        o.dist[row] = sqrt(best);
        o.cp[3 * (uint64_t)row] = cp.x;
        o.cp[3 * (uint64_t)row + 1] = cp.y;
        o.cp[3 * (uint64_t)row + 2] = cp.z;
        o.face[row] = bf;
        if (o.miss && table_miss(p, s, q, best, bf)) o.miss[atomicAdd(o.miss_n, 1u)] = row;  // not a superset: fallback
        if (kCounters && o.per_query) {
            o.per_query[3 * (uint64_t)row] = end - beg;
            o.per_query[3 * (uint64_t)row + 1] = exact;
        }
    }
    if (kCounters && o.agg) {
        unsigned long long v0 = active ? (end - beg) : 0ull, v1 = active ? exact : 0u, v2 = passes, v3 = rare_iters;
        unsigned long long v4 = sbytes + ((active && bf != 0xffffffffu) ? 96ull : 0ull);  // + the epilogue's record
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
            v0 += __shfl_down_sync(0xffffffffu, v0, sh);
            v1 += __shfl_down_sync(0xffffffffu, v1, sh);
            v2 += __shfl_down_sync(0xffffffffu, v2, sh);
            v3 += __shfl_down_sync(0xffffffffu, v3, sh);
            v4 += __shfl_down_sync(0xffffffffu, v4, sh);
        }
        if (lane == 0) {
            atomicAdd(o.agg + 0, v0);
            atomicAdd(o.agg + 1, v1);
            atomicAdd(o.agg + 4, v2);
            atomicAdd(o.agg + 5, v3);
            atomicAdd(o.agg + 6, v4);
            atomicAdd(o.agg + 7, 1ull);
        }
    }
}


// ---- warp tiles with a queued exact path ------------------------------------------------------
// Same tile walk as k_scan_small (windows of chunks, level-0/1 votes, best-first order, level-2 masks),
// but the exact evaluations are not done batch by batch by "the lanes whose bit is set" -- on c5 that
// runs the fp64 point-triangle kernel with ~4 of 32 lanes busy (profiles/r02).  Instead every
// (row, face) pair that passes level 2 is appended to a per-warp queue in shared memory, and whenever
// 32 pairs are queued the warp evaluates them one pair per lane, all lanes busy.  Each row's running
// (d^2 bits, face id) minimum lives in shared memory; a round merges into it with two atomicMin steps
// (d^2 first; then, among the pairs that attain the row's new d^2 -- plus the old face if d^2 did not
// change -- the lowest face id): the lexicographic argmin, whatever the evaluation order.  Pairs wait
// in the queue with the d_min of the moment they passed, which is only ever looser than the current
// one: a queued face may be evaluated needlessly, never skipped wrongly.
struct WarpQ {
    float4 row[32];                              // the tile's rows (fp32) and their squared bounds: group votes
    double qx[32], qy[32], qz[32];               // the tile's rows (fp64)
    unsigned long long best[32];                 // per row: bits of the smallest d^2 so far (+inf = none)
    uint32_t bf[32];                             // ... and its face (lowest id among ties)
    uint32_t ex[32];                             // per-row exact evaluations (counters mode)
    uint32_t qf[64];                             // queue: face id ...
    uint8_t qr[64];                              // ... and row lane of each waiting pair
};

template <bool kCounters>
__global__ void __launch_bounds__(256, P2M_SMALL_MINB) k_scan_warpq(Params p, const double* __restrict__ q_xyz,
                                                        const uint32_t* __restrict__ rows,
                                                        const uint32_t* __restrict__ key,
                                                        const uint32_t* __restrict__ tiles,
                                                        const uint32_t* __restrict__ meta,
                                                        const uint32_t* __restrict__ order, Out o) {
    __shared__ float4 s_disk[kWarps][64];
    __shared__ uint32_t s_fid[kWarps][32];
    __shared__ WarpQ s_wq[kWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t nt = meta[0], ns = meta[2];
    const uint32_t ti = blockIdx.x * kWarps + w;
    if (ti >= ns) return;                        // warp-uniform: no block barrier in this kernel
    float4* wd = s_disk[w];
    uint32_t* wf = s_fid[w];
    WarpQ& Q = s_wq[w];
    const uint32_t b = order[nt - ns + ti];
    const uint32_t start = tiles[b];
    const uint32_t stop = (b + 1 < nt) ? tiles[b + 1] : meta[1];
    const int m = (int)(stop - start);
    const uint32_t s = key[start];
    const bool active = lane < m;
    const float finf = __int_as_float(0x7f800000);
    uint32_t row = 0;
    float fx = 0.f, fy = 0.f, fz = 0.f;
    uint64_t DK = pk2(finf, finf);
    uint32_t exact_seed = 0;
    {
        V q{0, 0, 0};
        double best = __longlong_as_double(0x7ff0000000000000ll), dmin = best;
        uint32_t bf = 0xffffffffu;
        if (active) {
            row = rows[start + lane];
            q = V{q_xyz[3 * (uint64_t)row], q_xyz[3 * (uint64_t)row + 1], q_xyz[3 * (uint64_t)row + 2]};
            fx = (float)q.x; fy = (float)q.y; fz = (float)q.z;
            seed_row<kCounters>(p, s, q, pk2(fx, fx), pk2(fy, fy), pk2(fz, fz), dmin, DK, best, bf, exact_seed);
        }
        Q.qx[lane] = q.x; Q.qy[lane] = q.y; Q.qz[lane] = q.z;
        Q.best[lane] = (unsigned long long)__double_as_longlong(best);
        Q.bf[lane] = bf;
        if (kCounters) Q.ex[lane] = exact_seed;
        Q.row[lane] = make_float4(fx, fy, fz, 0.f);
    }
    __syncwarp();
    const float Mq = row_scale(p, fx, fy, fz);
    const float rx = __shfl_sync(0xffffffffu, fx, 0), ry = __shfl_sync(0xffffffffu, fy, 0),
                rz = __shfl_sync(0xffffffffu, fz, 0);  // the tile's first row: visiting order
    unsigned long long passes = 0, rare_iters = 0;
    unsigned long long sbytes = 0;               // structure bytes loaded (counters mode; bench roofline)
    const uint64_t beg = p.off[s], end = p.off[s + 1];
    const uint64_t bo = p.boff[s], co = p.coff[s];
    const uint32_t nch = (uint32_t)(p.coff[s + 1] - co);
    if (kCounters && lane == 0) sbytes += 16ull * nch + 76;  // chunk points, site ref, offsets, tile meta
    auto near = [&](float4 c0, float4 c1) {
        float dkx, dky;
        upk2(DK, dkx, dky);
        return cyl_near(fx, fy, fz, __fmul_ru(dkx, dkx), c0, c1);
    };
    auto bcast = [&](float4 v, int src) {
        return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                           __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
    };
    auto take_min = [&](uint32_t& k) {
        const uint32_t mk = __reduce_min_sync(0xffffffffu, k);
        const int src = __ffs(__ballot_sync(0xffffffffu, k == mk)) - 1;
        if (lane == src) k = 0xffffffffu;
        return src;
    };
    // the rows' current squared bounds for the transposed votes
    auto publish_bounds = [&]() {
        float dkx, dky;
        upk2(DK, dkx, dky);
        __syncwarp();
        Q.row[lane].w = __fmul_ru(dkx, dkx);
        __syncwarp();
    };
    uint32_t qhead = 0, qn = 0;                  // queue window [qhead, qhead + qn) mod 64 (warp-uniform)
    // one round: the first cnt (<= 32) queued pairs, one per lane, evaluated exactly and merged
    auto round = [&](uint32_t cnt) {
        const bool has = (uint32_t)lane < cnt;
        uint32_t f = 0;
        int r = 0;
        if (has) { f = Q.qf[(qhead + lane) & 63u]; r = Q.qr[(qhead + lane) & 63u]; }
        const unsigned long long old = Q.best[lane];
        const bool ev = has && f != Q.bf[r];     // the row's current face (the deep seed's) is done already
        unsigned long long kd = ~0ull;
        if (ev) {
            const V qr{Q.qx[r], Q.qy[r], Q.qz[r]};
            V a, b3, c3, pp3;
            load_tri(p.rec + 4 * (uint64_t)f, &a, &b3, &c3);
            kd = (unsigned long long)__double_as_longlong(closest_tri(qr, a, b3, c3, &pp3));  // d^2 >= +0: bits order as values
        }
        __syncwarp();                            // every lane has read old / bf before the merge
        if (ev) atomicMin(&Q.best[r], kd);
        __syncwarp();
        const unsigned long long nk = Q.best[lane];
        if (nk != old) Q.bf[lane] = 0xffffffffu; // a strictly smaller d^2: only its faces count
        __syncwarp();
        if (ev && kd == Q.best[r]) atomicMin(&Q.bf[r], f);
        if (kCounters) {
            if (ev) atomicAdd(&Q.ex[r], 1u);
            const uint32_t nev = __popc(__ballot_sync(0xffffffffu, ev));
            if (lane == 0) { rare_iters += 32; sbytes += 96ull * nev; }
        }
        __syncwarp();
        if (nk != old) {
            // any upper bound of sqrt(best) is a valid d_min: the fp32 sqrt rounded up of best rounded up
            const float dkf = dk_of(p, __fsqrt_ru(__double2float_ru(__longlong_as_double((long long)nk))), Mq);
            float dkx, dky;
            upk2(DK, dkx, dky);
            if (dkf < dkx) DK = pk2(dkf, dkf);
        }
        qhead = (qhead + cnt) & 63u;
        qn -= cnt;
    };
    float* wdf = reinterpret_cast<float*>(wd);
    for (uint32_t w0 = 0; w0 < nch; w0 += 32) {
        const int wn = (int)min(32u, nch - w0);
        float4 cc0 = make_float4(0.f, 0.f, 0.f, 0.f), cc1 = cc0;  // lane k: chunk w0 + k's cylinder
        if (lane < wn) { cc0 = p.ccy[kCy * (co + w0 + lane)]; cc1 = p.ccy[kCy * (co + w0 + lane) + 1]; }
        if (kCounters && lane == 0) sbytes += 32ull * wn;
        uint32_t cneed = 0;
        if (nch == 1 || p.no_batch) {
            cneed = wn == 32 ? 0xffffffffu : ((1u << wn) - 1u);
        } else if (p.tvote) {
            // transposed vote: lane k holds chunk k's cylinder and walks the tile's rows (shared memory,
            // broadcast reads) until one of them may need the chunk -- m row tests for the whole window
            // instead of a broadcast + test + vote per chunk; the same predicate on the same operands
            publish_bounds();
            bool need = false;
            if (lane < wn) {
                for (int r = 0; r < m; ++r) {
                    const float4 rw = Q.row[r];
                    if (cyl_near(rw.x, rw.y, rw.z, rw.w, cc0, cc1)) { need = true; break; }
                }
            }
            cneed = __ballot_sync(0xffffffffu, need);
        } else {
            for (int k = 0; k < wn; ++k) {
                const float4 c0 = bcast(cc0, k), c1 = bcast(cc1, k);
                if (__any_sync(0xffffffffu, active && near(c0, c1))) cneed |= 1u << k;
            }
        }
        const int nn = __popc(cneed);
        uint32_t ckey = ((cneed >> lane) & 1u) ? (nn > 1 ? cyl_key(rx, ry, rz, cc0, cc1) : 0u) : 0xffffffffu;
        for (int pos = 0; pos < nn; ++pos) {
            const int src = take_min(ckey);
            const uint32_t cidx = w0 + (uint32_t)src;
            if (pos > 0 && !p.no_batch) {
                const float4 c0 = bcast(cc0, src), c1 = bcast(cc1, src);
                if (!__any_sync(0xffffffffu, active && near(c0, c1))) continue;
            }
            const uint64_t cb = beg + (uint64_t)cidx * kChunk;
            const int nb = (int)((min((uint64_t)kChunk, end - cb) + 31) >> 5);
            if (kCounters && lane == 0) sbytes += 32ull * nb;
            float4 b0c = make_float4(0.f, 0.f, 0.f, 0.f), b1c = b0c;
            uint32_t bk = 0xffffffffu;
            if (lane < nb) {
                const uint64_t gi = kCy * (bo + (uint64_t)cidx * (kChunk / 32) + lane);
                b0c = p.bcy[gi];
                b1c = p.bcy[gi + 1];
                bk = nb > 1 ? cyl_key(rx, ry, rz, b0c, b1c) : 0u;
            }
            int nbv = nb;
            if (p.tvote && !p.no_batch) {
                // transposed pre-vote over the chunk's batches: lane L tests batch L & 7 against the rows
                // L >> 3, L >> 3 + 4, ...; a batch no row may need is never selected below
                publish_bounds();
                const float4 t0 = bcast(b0c, lane & 7), t1 = bcast(b1c, lane & 7);
                bool need = false;
                if ((lane & 7) < nb) {
                    for (int r = lane >> 3; r < m; r += 4) {
                        const float4 rw = Q.row[r];
                        if (cyl_near(rw.x, rw.y, rw.z, rw.w, t0, t1)) { need = true; break; }
                    }
                }
                uint32_t bn = __ballot_sync(0xffffffffu, need);
                bn = (bn | (bn >> 8) | (bn >> 16) | (bn >> 24)) & 0xffu;
                if (!((bn >> lane) & 1u)) bk = 0xffffffffu;
                nbv = __popc(bn);
            }
            for (int bpos = 0; bpos < nbv; ++bpos) {
                const int bsrc = take_min(bk);
                if (!p.no_batch && !(p.tvote && bpos == 0)) {   // (the pre-vote just held for the first one)
                    const float4 c0 = bcast(b0c, bsrc), c1 = bcast(b1c, bsrc);
                    if (!__any_sync(0xffffffffu, active && near(c0, c1))) continue;  // pruned whole
                }
                const uint64_t b0 = cb + 32ull * bsrc;
                const int valid = (int)min((uint64_t)32, end - b0);
                uint32_t f = 0;
                float4 r0 = kPadDisk, r1 = make_float4(0.f, 0.f, 0.f, 0.f);
                if (lane < valid) { f = p.lfs[b0 + lane]; r0 = p.fcy[kCy * (uint64_t)f]; r1 = p.fcy[kCy * (uint64_t)f + 1]; }
                wf[lane] = f;
                stage_disk(wdf, lane, r0, r1);
                __syncwarp();
                if (kCounters && lane == 0) sbytes += 36ull * valid;  // staged ids + disks
                uint32_t mask = batch_mask_row(p, active, pk2(fx, fx), pk2(fy, fy), pk2(fz, fz), DK, wd, valid, nullptr);
                if (kCounters) passes += __popc(mask);
                // Dense batch -- the rows want the same faces (a flat distance field: c3's cylinder axis,
                // where ~25 rows share each candidate): walk the union of the masks instead, so that one
                // broadcast read of a face record serves every row that needs it.  Queued, those pairs
                // would gather one record per lane (c3: 10.6 kB of records per query against 0.9, and
                // half the rate).  Sparse batches (c5: ~4 rows per candidate) go to the queue.
                {
                    uint32_t um = __reduce_or_sync(0xffffffffu, mask);
                    const uint32_t npairs = __reduce_add_sync(0xffffffffu, __popc(mask));
                    if (npairs >= p.dense_pairs * __popc(um) && um) {
                        if (kCounters && lane == 0) rare_iters += 32u * __popc(um);
                        while (um) {
                            const int kk = __ffs(um) - 1;
                            um &= um - 1;
                            bool ex = false;
                            if ((mask >> kk) & 1u) {
                                float dkx, dky;
                                upk2(DK, dkx, dky);
                                float4 r0, r1;
                                staged_disk(wdf, kk, r0, r1);
                                const uint32_t f = wf[kk];
                                if (cyl_near(fx, fy, fz, __fmul_ru(dkx, dkx), r0, r1) && f != Q.bf[lane]) {
                                    const V qr{Q.qx[lane], Q.qy[lane], Q.qz[lane]};
                                    V a, b3, c3, pp3;
                                    load_tri(p.rec + 4 * (uint64_t)f, &a, &b3, &c3);
                                    const double dd = closest_tri(qr, a, b3, c3, &pp3);
                                    const double best = __longlong_as_double((long long)Q.best[lane]);
                                    ex = true;
                                    if (kCounters) ++Q.ex[lane];
                                    if (dd < best || (dd == best && f < Q.bf[lane])) {   // this lane owns its row's slots
                                        Q.best[lane] = (unsigned long long)__double_as_longlong(dd);
                                        Q.bf[lane] = f;
                                        const float dkf = dk_of(p, __fsqrt_ru(__double2float_ru(dd)), Mq);
                                        if (dkf < dkx) DK = pk2(dkf, dkf);
                                    }
                                }
                            }
                            if (kCounters && __any_sync(0xffffffffu, ex) && lane == 0) sbytes += 96;
                        }
                        mask = 0u;
                    }
                }
                // append this batch's (row, face) pairs to the queue, in lane order, as many as fit; a
                // full warp's worth is evaluated as soon as it is there
                while (__any_sync(0xffffffffu, mask != 0u)) {
                    // exclusive prefix of the lanes' pair counts by bit planes (counts are small: one or
                    // two ballots instead of a five-step shuffle scan)
                    const uint32_t cnt = __popc(mask);
                    const uint32_t planes = __reduce_or_sync(0xffffffffu, cnt);
                    const uint32_t lt = (1u << lane) - 1u;
                    uint32_t wpos = 0, total = 0;
                    for (uint32_t bit = 1u; bit <= planes; bit <<= 1) {
                        if (!(planes & bit)) continue;
                        const uint32_t bl = __ballot_sync(0xffffffffu, (cnt & bit) != 0u);
                        wpos += bit * __popc(bl & lt);
                        total += bit * __popc(bl);
                    }
                    const uint32_t space = 64u - qn;
                    while (mask && wpos < space) {
                        const int k = __ffs(mask) - 1;
                        mask &= mask - 1;
                        const uint32_t slot = (qhead + qn + wpos) & 63u;
                        Q.qf[slot] = wf[k];
                        Q.qr[slot] = (uint8_t)lane;
                        ++wpos;
                    }
                    qn += min(total, space);
                    __syncwarp();
                    while (qn >= 32u) round(32u);
                }
                __syncwarp();                    // the slice is rewritten by the next batch
            }
        }
    }
    if (qn) round(qn);
    __syncwarp();
    if (active) {
        const V q{Q.qx[lane], Q.qy[lane], Q.qz[lane]};
        const double best = __longlong_as_double((long long)Q.best[lane]);
        const uint32_t bf = Q.bf[lane];
        V cp{__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll),
             __longlong_as_double(0x7ff8000000000000ll)};
        if (bf != 0xffffffffu) {
            V a, bb, c;
            load_tri(p.rec + 4 * (uint64_t)bf, &a, &bb, &c);
            closest_tri(q, a, bb, c, &cp);
        }
        o.dist[row] = sqrt(best);
        o.cp[3 * (uint64_t)row] = cp.x;
        o.cp[3 * (uint64_t)row + 1] = cp.y;
        o.cp[3 * (uint64_t)row + 2] = cp.z;
        o.face[row] = bf;
        if (o.miss && table_miss(p, s, q, best, bf)) o.miss[atomicAdd(o.miss_n, 1u)] = row;  // not a superset: fallback
        if (kCounters && o.per_query) {
            o.per_query[3 * (uint64_t)row] = end - beg;
            o.per_query[3 * (uint64_t)row + 1] = Q.ex[lane];
        }
    }
    if (kCounters && o.agg) {
        unsigned long long v0 = active ? (end - beg) : 0ull, v1 = active ? Q.ex[lane] : 0u, v2 = passes, v3 = rare_iters;
        unsigned long long v4 = sbytes + ((active && Q.bf[lane] != 0xffffffffu) ? 96ull : 0ull);  // + the epilogue's record
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
            v0 += __shfl_down_sync(0xffffffffu, v0, sh);
            v1 += __shfl_down_sync(0xffffffffu, v1, sh);
            v2 += __shfl_down_sync(0xffffffffu, v2, sh);
            v3 += __shfl_down_sync(0xffffffffu, v3, sh);
            v4 += __shfl_down_sync(0xffffffffu, v4, sh);
        }
        if (lane == 0) {
            atomicAdd(o.agg + 0, v0);
            atomicAdd(o.agg + 1, v1);
            atomicAdd(o.agg + 4, v2);
            atomicAdd(o.agg + 5, v3);
            atomicAdd(o.agg + 6, v4);
            atomicAdd(o.agg + 7, 1ull);
        }
    }
}


#ifndef P2M_EARLY1
#define P2M_EARLY1 1  // single-chunk CTA tiles: chunk loads issued before the seeds (cp.async batch cylinders)
#endif
#ifndef P2M_BATCH_ORDER
#define P2M_BATCH_ORDER 1   // block path: visit a chunk's batches best-first for the tile's first row
#endif
#ifndef P2M_SCAN_MINB
#define P2M_SCAN_MINB 4  // resident CTAs per SM the register budget is sized for
#endif
template <bool kCounters>
__global__ void __launch_bounds__(kTile, P2M_SCAN_MINB) k_scan_tiles(Params p, const double* __restrict__ q_xyz,
                                                         const uint32_t* __restrict__ rows,
                                                         const uint32_t* __restrict__ key,
                                                         const uint32_t* __restrict__ tiles,
                                                         const uint32_t* __restrict__ meta,
                                                         const uint32_t* __restrict__ order, Out o) {
    __shared__ float4 s_disk[2 * kChunk];        // the chunk's face disks, pair-interleaved (stage_disk)
    __shared__ uint32_t s_fid[kChunk];
    __shared__ float4 s_bcy[kCy * (kChunk / 32)];  // the chunk's batch cylinders
    __shared__ uint32_t s_need;                  // batches some warp of the CTA must scan
    __shared__ uint32_t s_cw[kWinChunks / 32];   // chunks of the current window some row must scan
    __shared__ uint32_t s_oidx[kWinChunks];      // ... in visiting order
    __shared__ uint32_t s_okey[kWinChunks];
    __shared__ float4 s_qrep;                    // the tile's first row (fp32), for the visiting order
    __shared__ uint32_t s_next;                  // small tiles: next batch of the window to scan
    __shared__ uint8_t s_bord[kChunk / 32];      // block path: visiting order of the chunk's batches
    __shared__ double s_rd[kTile];
    __shared__ uint32_t s_rf[kTile];
    __shared__ uint32_t s_re[kTile];
    __shared__ float s_dk[kTile];                // per row: the tightest d_min bound any replica found
    const uint32_t nt = meta[0];
    if (blockIdx.x >= nt - meta[2]) return;     // invalid, or a small tile (k_scan_small)
    const uint32_t b = order[blockIdx.x];        // launch order: site order or longest-first
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t start = tiles[b];
    const uint32_t stop = (b + 1 < nt) ? tiles[b + 1] : meta[1];
    const int m = (int)(stop - start);
    const uint32_t s = key[start];
    const long long t_start = p.tile_trace ? clock64() : 0;
    const int G = (m + 31) >> 5;
    const int R = max(1, kWarps / G);
    const int r = w / G;                         // replica of this warp (uniform per warp)
    const int j = (w % G) * 32 + lane;
    const bool warp_on = r < R;
    const bool active = warp_on && j < m;
    uint32_t row = 0;
    V q{0, 0, 0};
    uint64_t QX = 0, QY = 0, QZ = 0;
    if (active) {
        row = rows[start + j];
        q = V{q_xyz[3 * (uint64_t)row], q_xyz[3 * (uint64_t)row + 1], q_xyz[3 * (uint64_t)row + 2]};
        const float fx = (float)q.x, fy = (float)q.y, fz = (float)q.z;
        QX = pk2(fx, fx); QY = pk2(fy, fy); QZ = pk2(fz, fz);
        if (tid == 0) s_qrep = make_float4(fx, fy, fz, 0.f);
    }
    const float finf = __int_as_float(0x7f800000);
    double best = __longlong_as_double(0x7ff0000000000000ll), dmin = best;
    uint64_t DK = pk2(finf, finf);               // dk_of(upper bound of the row's distance), both halves
    uint32_t bf = 0xffffffffu;
    uint32_t exact = 0;
    unsigned long long passes = 0, rare_iters = 0;  // diagnostics (counters mode only)
    unsigned long long sbytes = 0;               // structure bytes loaded (counters mode; bench roofline)
    const uint64_t beg = p.off[s], end = p.off[s + 1];
    float* s_df = reinterpret_cast<float*>(s_disk);
    const uint64_t bo = p.boff[s];               // this list's first 32-entry batch
    const uint64_t co = p.coff[s];               // ... and first 256-entry chunk
    const uint32_t nch = (uint32_t)(p.coff[s + 1] - co);
    if (kCounters && tid == 0) sbytes += 48ull * nch + 76;  // chunk spheres + cylinders, site ref, offsets, tile meta
#define qxf __uint_as_float((uint32_t)QX)
#define qyf __uint_as_float((uint32_t)QY)
#define qzf __uint_as_float((uint32_t)QZ)
    // register prefetch of one chunk entry per thread: face id + its disk record
    uint32_t nf = 0;
    float4 nv0 = kPadDisk, nv1 = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t pre_c = 0xffffffffu;                // chunk held in (nf, nv0, nv1)
    bool first_chunk = true;
#if P2M_EARLY1
    const bool early = nch == 1 && G > 1;        // the one chunk of a single-chunk CTA tile: its loads
    if (early) {                                 // start now and land during the seed computation
        const int mc0 = (int)min((uint64_t)kChunk, end - beg);
        if (tid < kCy * ((mc0 + 31) >> 5)) {     // batch cylinders: async copy to shared, no registers
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&s_bcy[tid]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(p.bcy + kCy * bo + tid));
        }
        asm volatile("cp.async.commit_group;");
        if (tid < mc0) { nf = p.lfs[beg + tid]; nv0 = p.fcy[kCy * (uint64_t)nf]; nv1 = p.fcy[kCy * (uint64_t)nf + 1]; }
        pre_c = 0;
    }
#endif
    if (active) seed_row<kCounters>(p, s, q, QX, QY, QZ, dmin, DK, best, bf, exact);
    if (active && r == 0) {                      // replicas share one pruning bound per row
        float dkx, dky;
        upk2(DK, dkx, dky);
        s_dk[j] = dkx;
    }
    auto refresh_dk = [&]() {                    // the row's bound as tightened by the other replicas
        if (R > 1 && active) {
            float dkx, dky;
            upk2(DK, dkx, dky);
            const float v = s_dk[j];
            if (v < dkx) DK = pk2(v, v);
        }
    };
    auto near = [&](float4 c0, float4 c1) {      // conservative: may a member of the group be within d_min?
        float dkx, dky;
        upk2(DK, dkx, dky);
        return cyl_near(qxf, qyf, qzf, __fmul_ru(dkx, dkx), c0, c1);
    };
    for (uint32_t w0 = 0; w0 < nch; w0 += kWinChunks) {
        const uint32_t wn = min(nch - w0, (uint32_t)kWinChunks);
        const int nwords = (int)((wn + 31) >> 5);
        // level 0: a chunk is scanned only if some row's conservative bound to its cylinder does not
        // exceed that row's d_min (any replica's d_min is a valid upper bound of the row's distance)
        // a single-chunk list (most tiles) has a trivial window: no votes, no ordering, no barriers
        int nord = 1;
        if (nch > 1) {
            if (w0 != 0) __syncthreads();            // every thread is done with the previous window's order
            if (tid < kWinChunks / 32) {
                const int nv_ = min(32, max(0, (int)wn - 32 * tid));
                const uint32_t vmask = nv_ == 32 ? 0xffffffffu : ((1u << nv_) - 1u);
                s_cw[tid] = p.no_batch ? vmask : 0u;
            }
            __syncthreads();
            if (warp_on && !p.no_batch) {
                for (int wi = r; wi < nwords; wi += R) {
                    uint32_t bits = 0;
                    const int kn = min(32, (int)wn - 32 * wi);
                    for (int k = 0; k < kn; ++k) {
                        const uint64_t gi = kCy * (co + w0 + 32 * wi + k);
                        const bool need = active && near(p.ccy[gi], p.ccy[gi + 1]);
                        if (__any_sync(0xffffffffu, need)) bits |= 1u << k;
                    }
                    if (lane == 0 && bits) atomicOr(&s_cw[wi], bits);
                }
            }
            __syncthreads();
            // Visit the needed chunks best-first for the tile's first row (every row of the tile lies in
            // the same Voronoi cell): an early small d_min then prunes most later chunks at the batch
            // level.  The order changes neither the (d^2, face id) argmin nor which faces may be skipped.
            {
                int pos = -1;
                uint32_t okey = 0;
                if (tid < (int)wn) {
                    const uint32_t wb = s_cw[tid >> 5];
                    if ((wb >> (tid & 31)) & 1u) {
                        pos = __popc(wb & ((1u << (tid & 31)) - 1u));
                        for (int k = 0; k < (tid >> 5); ++k) pos += __popc(s_cw[k]);
                        const uint64_t gi = kCy * (co + w0 + tid);
                        const float4 qr = s_qrep;
                        okey = cyl_key(qr.x, qr.y, qr.z, p.ccy[gi], p.ccy[gi + 1]);
                    }
                }
                nord = 0;
                for (int k = 0; k < nwords; ++k) nord += __popc(s_cw[k]);
                if (pos >= 0) { s_oidx[pos] = (uint32_t)tid; s_okey[pos] = okey; }
                __syncthreads();
                if (nord > 1) {
                    uint32_t mi = 0, rank = 0;
                    if (tid < nord) {
                        mi = s_oidx[tid];
                        const uint32_t mk = s_okey[tid];
                        for (int u = 0; u < nord; ++u) {
                            const uint32_t ku = s_okey[u];
                            rank += (ku < mk || (ku == mk && u < tid)) ? 1u : 0u;
                        }
                    }
                    __syncthreads();
                    if (tid < nord) s_oidx[rank] = mi;
                    __syncthreads();
                }
            }
        }
        auto scan_batch = [&](const float4* disk, const uint32_t* fid, int valid) {
            scan_batch_row<kCounters>(p, active, q, QX, QY, QZ, DK, best, bf, exact, passes, rare_iters, sbytes,
                                      disk, fid, valid, lane, R > 1 && active ? &s_dk[j] : nullptr);
        };
        if (G == 1) {
            // Small tile (<= 32 rows): every warp holds all rows, so each batch needs only one warp.
            // Warps pull batches of the ordered chunks from a shared counter and stage them in their
            // own shared-memory slice -- no block barrier until the window ends, and the load
            // balances itself (replica warps otherwise wait at every chunk for the slowest one).
            if (tid == 0) s_next = 0u;
            __syncthreads();
            const uint32_t T = (uint32_t)nord * (kChunk / 32);
            float4* wd = s_disk + 64 * w;
            float* wdf = reinterpret_cast<float*>(wd);
            uint32_t* wf = s_fid + 32 * w;
            for (;;) {
                uint32_t t = 0;
                if (lane == 0) t = atomicAdd(&s_next, 1u);
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t >= T) break;
                const uint32_t cidx = w0 + (nch > 1 ? s_oidx[t / (kChunk / 32)] : 0u);
                const uint32_t gb = cidx * (kChunk / 32) + t % (kChunk / 32);  // batch index in the list
                const uint64_t b0 = beg + 32ull * gb;
                if (b0 >= end) continue;
                const int valid = (int)min((uint64_t)32, end - b0);
                bool need = p.no_batch != 0;
                refresh_dk();
                if (active && !need) need = near(p.bcy[kCy * (bo + gb)], p.bcy[kCy * (bo + gb) + 1]);
                if (kCounters && lane == 0) sbytes += 32;  // the batch cylinder
                if (!__any_sync(0xffffffffu, need)) continue;  // pruned whole by its batch cylinder
                if (kCounters && lane == 0) sbytes += 36ull * valid;  // staged ids + disks
                uint32_t f = 0;
                float4 r0 = kPadDisk, r1 = make_float4(0.f, 0.f, 0.f, 0.f);
                if (lane < valid) { f = p.lfs[b0 + lane]; r0 = p.fcy[kCy * (uint64_t)f]; r1 = p.fcy[kCy * (uint64_t)f + 1]; }
                wf[lane] = f;
                stage_disk(wdf, lane, r0, r1);
                __syncwarp();
                scan_batch(wd, wf, valid);
                __syncwarp();                    // the slice is rewritten by the next batch
            }
            continue;                            // next window (its first barrier orders s_next)
        }
        for (int oi = 0; oi < nord; ++oi) {
            const uint32_t cidx = w0 + (nch > 1 ? s_oidx[oi] : 0u);
            const uint64_t base = beg + (uint64_t)cidx * kChunk;
            const int mc = (int)min((uint64_t)kChunk, end - base);
            const int nb = (mc + 31) >> 5;
            if (!first_chunk) __syncthreads();   // the previous chunk is fully consumed
            first_chunk = false;
            if (pre_c != cidx) {
                nf = 0;
                nv0 = kPadDisk;
                nv1 = make_float4(0.f, 0.f, 0.f, 0.f);
                if (tid < mc) { nf = p.lfs[base + tid]; nv0 = p.fcy[kCy * (uint64_t)nf]; nv1 = p.fcy[kCy * (uint64_t)nf + 1]; }
            }
            // level 1: the enclosing cylinder of each 32-entry batch.  If every lane's conservative
            // bound to it exceeds the lane's d_min, every member face's bound does too, so the whole
            // batch is pruned exactly as the per-candidate tests would prune it (and is never staged).
#if P2M_EARLY1
            if (early) {
                asm volatile("cp.async.wait_all;" ::: "memory");
            } else if (tid < kCy * nb) {
                s_bcy[tid] = p.bcy[kCy * (bo + (uint64_t)cidx * (kChunk / 32)) + tid];
            }
#else
            if (tid < kCy * nb) s_bcy[tid] = p.bcy[kCy * (bo + (uint64_t)cidx * (kChunk / 32)) + tid];
#endif
            if (tid == 0) s_need = 0u;
            __syncthreads();
            uint32_t wneed = 0;
            refresh_dk();
            if (warp_on) {
                for (int bb = r; bb < nb; bb += R) {
                    bool need = p.no_batch != 0;
                    if (active && !need) need = near(s_bcy[kCy * bb], s_bcy[kCy * bb + 1]);
                    if (__any_sync(0xffffffffu, need)) wneed |= 1u << bb;
                }
                if (lane == 0 && wneed) atomicOr(&s_need, wneed);
            }
            __syncthreads();
            const uint32_t cneed = s_need;
            if (kCounters && tid == 0) {         // ids + disks of the needed batches, batch cylinders
                sbytes += 32ull * nb;
                for (int bb = 0; bb < nb; ++bb)
                    if ((cneed >> bb) & 1u) sbytes += 36ull * min(32, mc - 32 * bb);
            }
            // prefetch the window's next chunk while this one is scanned
            auto prefetch_next = [&]() {
                pre_c = 0xffffffffu;
                if (oi + 1 < nord) {
                    const uint32_t c2 = w0 + (nch > 1 ? s_oidx[oi + 1] : 0u);
                    const uint64_t b2 = beg + (uint64_t)c2 * kChunk;
                    nf = 0;
                    nv0 = kPadDisk;
                    nv1 = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (b2 + tid < end) { nf = p.lfs[b2 + tid]; nv0 = p.fcy[kCy * (uint64_t)nf]; nv1 = p.fcy[kCy * (uint64_t)nf + 1]; }
                    pre_c = c2;
                }
            };
            if (!cneed) {                        // every batch pruned with the current d_min
                prefetch_next();
                continue;
            }
            if (P2M_BATCH_ORDER && w == 0) {
                // the chunk's batches best-first for the tile's first row (all rows share a cell)
                uint32_t bkey = 0xffffffffu;
                if (lane < nb) {
                    const float4 qr = s_qrep;
                    bkey = cyl_key(qr.x, qr.y, qr.z, s_bcy[kCy * lane], s_bcy[kCy * lane + 1]);
                }
                uint32_t rk = 0;
#pragma unroll
                for (int jj = 0; jj < kChunk / 32; ++jj) {
                    const uint32_t kj = __shfl_sync(0xffffffffu, bkey, jj);
                    rk += (kj < bkey || (kj == bkey && jj < lane)) ? 1u : 0u;
                }
                if (lane < nb) s_bord[rk] = (uint8_t)lane;
            }
            if ((cneed >> (tid >> 5)) & 1u) {    // stage the needed batches: face ids + disks
                s_fid[tid] = nf;
                stage_disk(s_df, tid, nv0, nv1);
            }
            __syncthreads();
            prefetch_next();
            if (!warp_on) continue;
            for (int pos = r; pos < nb; pos += R) {
                const int bb = P2M_BATCH_ORDER ? (int)s_bord[pos] : pos;
                // pruned whole by its batch cylinder for every row (cneed: the union over the replicas'
                // level-1 votes -- with the reordering a replica scans batches another one voted on).
                // Without replicas each warp voted on every batch for its own rows: a batch its own
                // vote pruned stays pruned (d_min only shrinks), so it is skipped too.
                if (!(((R == 1 ? wneed : cneed) >> bb) & 1u)) continue;
                scan_batch(s_disk + 64 * bb, s_fid + 32 * bb, mc - 32 * bb);
            }
        }
    }
#undef qxf
#undef qyf
#undef qzf
    if (R > 1) {
        __syncthreads();
        const int slot = r * G * 32 + j;
        if (active) { s_rd[slot] = best; s_rf[slot] = bf; s_re[slot] = exact; }
        __syncthreads();
        if (active && r == 0) {
            for (int rr = 1; rr < R; ++rr) {
                const int o2 = rr * G * 32 + j;
                const double d2 = s_rd[o2];
                const uint32_t f2 = s_rf[o2];
                if (d2 < best || (d2 == best && f2 < bf)) { best = d2; bf = f2; }
                exact += s_re[o2];
            }
        }
    }
    if (p.tile_trace && tid == 0) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* t = p.tile_trace + 4 * (uint64_t)b;
        t[0] = s; t[1] = (unsigned long long)m; t[2] = p.off[s + 1] - p.off[s];
        t[3] = (unsigned long long)(clock64() - t_start) << 8 | (smid & 0xff);
    }
    const bool writer = active && r == 0;
    if (writer) {
        V cp{__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll),
             __longlong_as_double(0x7ff8000000000000ll)};
        if (bf != 0xffffffffu) {
            V a, bb, c;
            load_tri(p.rec + 4 * (uint64_t)bf, &a, &bb, &c);
            closest_tri(q, a, bb, c, &cp);
        }
        o.dist[row] = sqrt(best);
        o.cp[3 * (uint64_t)row] = cp.x;
        o.cp[3 * (uint64_t)row + 1] = cp.y;
        o.cp[3 * (uint64_t)row + 2] = cp.z;
        o.face[row] = bf;
        if (o.miss && table_miss(p, s, q, best, bf)) o.miss[atomicAdd(o.miss_n, 1u)] = row;  // not a superset: fallback
        if (kCounters && o.per_query) {
            o.per_query[3 * (uint64_t)row] = end - beg;
            o.per_query[3 * (uint64_t)row + 1] = exact;
        }
    }
    if (kCounters && o.agg) {
        unsigned long long v0 = writer ? (end - beg) : 0ull, v1 = writer ? exact : 0u;
        unsigned long long v2 = passes, v3 = rare_iters;
        unsigned long long v4 = sbytes + ((writer && bf != 0xffffffffu) ? 96ull : 0ull);  // + the epilogue's record
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
            v2 += __shfl_down_sync(0xffffffffu, v2, sh);
            v3 += __shfl_down_sync(0xffffffffu, v3, sh);
            v4 += __shfl_down_sync(0xffffffffu, v4, sh);
        }
        if (lane == 0) {
            atomicAdd(o.agg + 4, v2);
            atomicAdd(o.agg + 5, v3);
            atomicAdd(o.agg + 6, v4);
        }
        if (tid == 0) atomicAdd(o.agg + 7, 1ull);
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) {
            v0 += __shfl_down_sync(0xffffffffu, v0, sh);
            v1 += __shfl_down_sync(0xffffffffu, v1, sh);
        }
        if (lane == 0) {
            atomicAdd(o.agg + 0, v0);
            atomicAdd(o.agg + 1, v1);
        }
    }
}


}  // namespace

// Rows of a table miss (the scan kept no face: every list face lay beyond the row's d_min seed, which
// only happens if the list is not a Theorem-1 superset): the exact BVH closest point over all faces
// (REF/SPEC.md:201-209), flagged P2M_FLAG_FALLBACK | P2M_FLAG_TABLE_MISS.  Never fires on tables the
// builder produced; one tiny launch per query.
__global__ void __launch_bounds__(128) k_table_miss(Params p, const double* __restrict__ q_xyz, Out o) {
    const uint32_t cnt = *o.miss_n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const uint32_t row = o.miss[i];
        const V q{q_xyz[3 * (uint64_t)row], q_xyz[3 * (uint64_t)row + 1], q_xyz[3 * (uint64_t)row + 2]};
        double best;
        const uint32_t bf = bvh_closest(p, q, &best);
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
        if (o.flags) o.flags[row] |= 5u;         // P2M_FLAG_FALLBACK | P2M_FLAG_TABLE_MISS
    }
}

cudaError_t launch_table_miss(const Params& p, const double* q, const Out& o, cudaStream_t s) {
    if (!o.miss) return cudaSuccess;
    k_table_miss<<<2 * 148, 128, 0, s>>>(p, q, o);
    return cudaGetLastError();
}

cudaError_t launch_descend(const Params& p, const double* q, const uint32_t* rows, uint64_t n, uint32_t* site_key,
                           const Out& o, bool counters, cudaStream_t s) {
    if (!n) return cudaSuccess;
    const unsigned g = (unsigned)((n + 255) / 256);
    if (counters) k_descend<true><<<g, 256, 0, s>>>(p, q, rows, n, site_key, o);
    else k_descend<false><<<g, 256, 0, s>>>(p, q, rows, n, site_key, o);
    return cudaGetLastError();
}

struct MaxU32 {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};
static cudaError_t scan_max_u32(void* tmp, size_t& bytes, const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
    return cub::DeviceScan::InclusiveScan(tmp, bytes, in, out, MaxU32{}, (int64_t)n, s);
}
static cudaError_t scan_sum_u32(void* tmp, size_t& bytes, const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
    return cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int64_t)n, s);
}

size_t tiles_tmp_bytes(uint64_t n) {
    size_t a = 0, b = 0;
    scan_max_u32(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0);
    scan_sum_u32(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, n, 0);
    return std::max(a, b);
}

cudaError_t launch_tiles(const Params& p, const uint32_t* key, uint64_t n, uint32_t n_sites, uint32_t* hpos, uint32_t* run_start,
                         uint32_t* flag, uint32_t* tix, uint32_t* tiles, uint32_t* meta, void* tmp, size_t tmp_bytes,
                         cudaStream_t s) {
    if (!n) return cudaSuccess;
    const unsigned g = (unsigned)((n + 255) / 256);
    cudaError_t e;
    k_run_heads<<<g, 256, 0, s>>>(key, n, hpos);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    size_t tb = tmp_bytes;
    if ((e = scan_max_u32(tmp, tb, hpos, run_start, n, s)) != cudaSuccess) return e;
    k_tile_flags<<<g, 256, 0, s>>>(p, key, run_start, n, n_sites, flag, meta);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    tb = tmp_bytes;
    if ((e = scan_sum_u32(tmp, tb, flag, tix, n, s)) != cudaSuccess) return e;
    k_tile_write<<<g, 256, 0, s>>>(flag, tix, n, tiles, meta);
    return cudaGetLastError();
}

uint64_t max_tiles(uint64_t n, uint64_t n_sites) { return std::min<uint64_t>(n, n_sites) + (n + 31) / 32 + 1; }

// Longest-processing-time-first launch order of the tiles: a tile's time grows with its list
// length and, more weakly, with its rows, and the heaviest tiles (long auxiliary lists) sit at the
// END of the site-sorted order -- launched last, they would set a tail of up to ~2.5 ms on c2.
__global__ void __launch_bounds__(256) k_tile_keys(Params p, const uint32_t* __restrict__ key,
                                                   const uint32_t* __restrict__ tiles,
                                                   uint32_t* __restrict__ meta, uint32_t max_t,
                                                   uint32_t* __restrict__ tkey, uint32_t* __restrict__ tidx) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nt = meta[0];
    uint32_t k = 0;
    bool small = false;
    if (t < nt) {
        const uint32_t start = tiles[t];
        const uint32_t stop = (t + 1 < nt) ? tiles[t + 1] : meta[1];
        const uint32_t s = key[start];
        const uint64_t len0 = p.off[s + 1] - p.off[s];
        const uint64_t len = len0 < (1u << 20) ? len0 : (1u << 20);
        const uint64_t nch = p.coff[s + 1] - p.coff[s];
        small = p.warp_tiles || (stop - start <= 32u && (nch <= p.small_chunks ||
                                 (p.warp_min_chunks && nch >= p.warp_min_chunks && !p.heavy[s])));
        if (small && !p.warp_tiles) k = 1u;      // after every CTA tile: k_scan_small's range
        else if (p.tile_order == 1) k = (uint32_t)((len * (uint64_t)(stop - start + 16)) >> 4) + 2u;
        else if (p.tile_order == 2) k = (uint32_t)(64 - __clzll((long long)len)) + 2u;  // coarse buckets
        else k = 2u;                             // site order (the sort is stable)
    }  // invalid tiles keep 0: launched last (and exit at once)
    if (t < max_t) {
        tkey[t] = k;
        tidx[t] = t;
    }
    const uint32_t nsm = __popc(__ballot_sync(0xffffffffu, small));
    if ((threadIdx.x & 31) == 0 && nsm) atomicAdd(meta + 2, nsm);
}

size_t tile_order_tmp_bytes(uint64_t max_t) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                              (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)max_t, 0, 32, 0);
    return b;
}

cudaError_t launch_tile_order(const Params& p, const uint32_t* key, const uint32_t* tiles, uint32_t* meta,
                              uint64_t max_t, uint32_t* tkey, uint32_t* tkey2, uint32_t* tidx, uint32_t* order,
                              void* tmp, size_t tmp_bytes, cudaStream_t s) {
    if (!max_t) return cudaSuccess;
    k_tile_keys<<<(unsigned)((max_t + 255) / 256), 256, 0, s>>>(p, key, tiles, meta, (uint32_t)max_t, tkey, tidx);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    size_t tb = tmp_bytes;
    const int bits = p.tile_order == 1 ? 32 : p.tile_order == 2 ? 8 : 2;  // key ranges of k_tile_keys
    return cub::DeviceRadixSort::SortPairsDescending(tmp, tb, tkey, tkey2, tidx, order, (int64_t)max_t, 0, bits, s);
}

// the warp-tile kernel: queued exact path (default) or the batch-by-batch union walk (P2M_NO_WARP_QUEUE)
static void launch_warp_tiles(const Params& p, const double* q, const uint32_t* rows, const uint32_t* key,
                              const uint32_t* tiles, const uint32_t* meta, const uint32_t* order, const Out& o,
                              bool counters, unsigned gs, cudaStream_t s) {
    if (p.warp_queue) {
        if (counters) k_scan_warpq<true><<<gs, kTile, 0, s>>>(p, q, rows, key, tiles, meta, order, o);
        else k_scan_warpq<false><<<gs, kTile, 0, s>>>(p, q, rows, key, tiles, meta, order, o);
    } else {
        if (counters) k_scan_small<true><<<gs, kTile, 0, s>>>(p, q, rows, key, tiles, meta, order, o);
        else k_scan_small<false><<<gs, kTile, 0, s>>>(p, q, rows, key, tiles, meta, order, o);
    }
}

cudaError_t launch_scan_tiles(const Params& p, const double* q, const uint32_t* rows, const uint32_t* key,
                              const uint32_t* tiles, const uint32_t* meta, const uint32_t* order, uint64_t n,
                              const Out& o, bool counters, cudaStream_t s, cudaStream_t side, cudaEvent_t fork,
                              cudaEvent_t join) {
    if (!n) return cudaSuccess;
    if (!order) return cudaErrorInvalidValue;   // the launch order (launch_tile_order) is required
    const unsigned g = (unsigned)max_tiles(n, p.n_nodes);
    cudaError_t e;
    if (p.warp_tiles) {                          // warp mode: every tile is a warp tile
        const unsigned gs = (g + kWarps - 1) / kWarps;
        launch_warp_tiles(p, q, rows, key, tiles, meta, order, o, counters, gs, s);
        return cudaGetLastError();
    }
    // warp tiles (small lists, or every non-heavy site in sparse batches): k_scan_small, on a side
    // stream forked from and joined back to s when there is one, so it overlaps k_scan_tiles
    const bool small = p.small_chunks || p.warp_min_chunks;
    const bool fork_side = small && side;
    if (small) {
        cudaStream_t ss = s;
        if (fork_side) {
            if ((e = cudaEventRecord(fork, s)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(side, fork, 0)) != cudaSuccess) return e;
            ss = side;
        }
        const unsigned gs = (g + kWarps - 1) / kWarps;
        launch_warp_tiles(p, q, rows, key, tiles, meta, order, o, counters, gs, ss);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (fork_side && (e = cudaEventRecord(join, side)) != cudaSuccess) return e;
    }
    if (counters) k_scan_tiles<true><<<g, kTile, 0, s>>>(p, q, rows, key, tiles, meta, order, o);
    else k_scan_tiles<false><<<g, kTile, 0, s>>>(p, q, rows, key, tiles, meta, order, o);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (fork_side && (e = cudaStreamWaitEvent(s, join, 0)) != cudaSuccess) return e;  // join
    return cudaGetLastError();
}

}  // namespace dev
}  // namespace p2m
