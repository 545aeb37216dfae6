// p2m_device.cuh -- device-side data layout and fp64 primitives of the query path (sm_100a).
//
// Layout in HBM (one replica per GPU):
//   kd nodes   : double4[S]  {x, y, z, meta}  meta bits = site id (0..31) | split dim (32..33) |
//                sentinel (34); left-balanced k-d tree in BFS order, children 2k+1 / 2k+2
//   face recs  : double4[4F] one 128-byte line per face: {c.xyz, r}, {a.xyz, b.x}, {b.yz, c.xy},
//                {c.z, 0, 0, 0} -- the pruning sphere is the first 32-byte sector, the triangle the
//                next three, so an exact evaluation touches the line its sphere test already pulled
//   lists      : u64 offsets[S+1], u32 face ids (CSR, ascending per site)
//   bvh nodes  : double4[2 * nodes] fallback BVH {lo.xyz, hi.x}, {hi.yz, meta, 0}
// Every 32-byte record is fetched with one 256-bit load (LDG.E.ENL2.256).
//
// fp64 parity: the translation unit is compiled with --fmad=false and the operation order of
// REF/proj/src/geom.cpp:31-70 (dot = (x*x + y*y) + z*z, a + ab*v, (a + ab*v) + ac*w), so d^2, the
// closest point and the distance are bit-identical to the reference on the same inputs.
#pragma once

#include <cstdint>

namespace p2m {
namespace dev {

struct __align__(32) D4 {
    double x, y, z, w;
};

__device__ __forceinline__ D4 ldg4(const D4* p) {
    D4 r;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
                 : "l"(p));
    return r;
}

struct V {
    double x, y, z;
};
__device__ __forceinline__ V vsub(V a, V b) { return V{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double vdot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double vd2(V a, V b) { V d = vsub(a, b); return vdot(d, d); }
__device__ __forceinline__ V vaxpy(V a, V d, double s) { return V{a.x + d.x * s, a.y + d.y * s, a.z + d.z * s}; }

// Closest point on triangle (a,b,c) to q and its squared distance: REF/proj/src/geom.cpp:31-70.
__device__ __forceinline__ double closest_tri(V q, V a, V b, V c, V* pout) {
    const V ab = vsub(b, a), ac = vsub(c, a), aq = vsub(q, a);
    const double d1 = vdot(ab, aq), d2 = vdot(ac, aq);
    if (d1 <= 0.0 && d2 <= 0.0) { *pout = a; return vd2(q, a); }
    const V bq = vsub(q, b);
    const double d3 = vdot(ab, bq), d4 = vdot(ac, bq);
    if (d3 >= 0.0 && d4 <= d3) { *pout = b; return vd2(q, b); }
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        const double v = d1 / (d1 - d3);
        *pout = vaxpy(a, ab, v); return vd2(q, *pout);
    }
    const V cq = vsub(q, c);
    const double d5 = vdot(ab, cq), d6 = vdot(ac, cq);
    if (d6 >= 0.0 && d5 <= d6) { *pout = c; return vd2(q, c); }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const double w = d2 / (d2 - d6);
        *pout = vaxpy(a, ac, w); return vd2(q, *pout);
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        *pout = vaxpy(b, vsub(c, b), w); return vd2(q, *pout);
    }
    const double denom = 1.0 / (va + vb + vc);
    const double v = vb * denom, w = vc * denom;
    *pout = vaxpy(vaxpy(a, ab, v), ac, w);
    return vd2(q, *pout);
}

__device__ __forceinline__ void load_tri(const D4* rec, V* a, V* b, V* c) {
    const D4 t0 = ldg4(rec + 1), t1 = ldg4(rec + 2), t2 = ldg4(rec + 3);
    *a = V{t0.x, t0.y, t0.z};
    *b = V{t0.w, t1.x, t1.y};
    *c = V{t1.z, t1.w, t2.x};
}

constexpr int kCy = 2;      // float4 per bounding-cylinder record (Params::fcy / bcy / ccy)
constexpr uint64_t kIdMask = 0xffffffffull;
constexpr int kDimShift = 32;
constexpr uint64_t kSentinelBit = 1ull << 34;

struct Params {
    const D4* kd;           // S nodes
    uint32_t n_nodes;
    const D4* rec;          // 4 per face
    // bounding cylinders (kCy = 2 float4 each: {c.xyz, 4 R^2}, {n.xyz, t}; every point x of every member
    // face has |nn.(x - c)| <= t and in-plane distance <= R, nn = n / |n|; p2m_engine.cu fit_cyl):
    const float4* fcy;      // per face (its bounding disk: level 2 of the grouped scan)
    const float4* bcy;      // per aligned 32-entry batch of lfs (level 1)
    const float4* ccy;      // per aligned 256-entry chunk of lfs (level 0)
    const uint64_t* off;    // S+1
    const uint64_t* boff;   // S+1: first batch sphere of each list (one per aligned 32 entries of lfs)
    const float4* bpt;      // per batch: {a point ON the mesh near the batch centre (fp32), 0} -- d_min seeds
    const uint32_t* lf;     // list entries, ascending (REF/SPEC.md:392; the fused sequential path)
    const uint32_t* lfs;    // the same lists in spatial (Morton) order (the grouped scan)
    const uint64_t* coff;   // S+1: first chunk sphere of each list (one per aligned 256 entries of lfs)
    const float4* cpt;      // per chunk: the same for the chunk
    const D4* bvh;          // 2 per node
    const uint32_t* bvh_perm;  // leaf face ids
    uint32_t n_faces;
    double dmin[3], dmax[3];
    double prune_eps;
    double key_lo[3], key_scale[3];  // Morton key box
    float mesh_m;           // max |coordinate| of the mesh and of every stored centre / point (fp32 error scale)
    float eps2;             // 2 * prune_eps, rounded up
    float ctr_slack;        // max over faces of d(fp32 disk centre, face): |q - c| + this bounds d(q, face) from above
    const uint8_t* heavy;   // per site: 1 if its rows are tiled long_tile rows per CTA
    uint32_t long_tile;     // (32, 64, 128 or 256)
    // exact grid cell-locate (optional, grid_off == nullptr -> k-d tree only): every site whose
    // Voronoi cell box meets grid cell c is listed in grid_site[grid_off[c] .. grid_off[c+1])
    const D4* site_pos;     // by site id: {x, y, z, meta (sentinel bit)}
    const D4* site_ref;     // by site id: a point on the mesh {x, y, z, 1} or {.., .., .., 0} = none
    int no_seed;            // 0: every d_min seed; 1: d_min starts at +inf in the grouped scan too (P2M_NO_SEED);
                            // 2: group-point seeds only, no per-row exact seed face (P2M_NO_DEEP_SEED)
    int no_batch;           // 1: no level-1 batch-sphere pruning (P2M_NO_BATCH)
    const uint32_t* grid_off;
    const uint32_t* grid_site;
    int nns;                // P2M_NNS_* strategy of nearest_site
    int tile_order;         // scan launch order: 0 site order, 1 longest-first, 2 list-length buckets
    uint32_t small_chunks;  // tiles of <= 32 rows and lists of <= this many chunks: one warp per tile (0: off)
    int warp_tiles;         // 1: every tile has <= 32 rows and is scanned by one warp (k_scan_small); no k_scan_tiles
    int tvote;              // 1: k_scan_warpq votes on chunks / batches lane-parallel over the groups (P2M_NO_TVOTE: 0)
    uint32_t dense_pairs;   // k_scan_warpq: a batch whose rows average >= this many per wanted face walks the union
                            // of their masks (broadcast record reads) instead of queueing the pairs (P2M_DENSE_PAIRS)
    int warp_queue;         // 1: warp tiles queue their (row, face) pairs and evaluate 32 at a time (k_scan_warpq)
    uint32_t warp_min_chunks;  // sites (not heavy) whose list has >= this many chunks get 32-row warp tiles (0: off, ~0: auto)
    unsigned long long* tile_trace;  // debug (P2M_TILE_TRACE): per tile {site, rows, list length, cycles | sm}
    const uint64_t* adj_off;  // Delaunay adjacency CSR (nullptr: no DelaunayWalk)
    const uint32_t* adj;
    double grid_lo[3], grid_inv[3];
    uint32_t grid_res[3];
};

// Grid cell of q; false if q lies outside the grid box (the caller then uses the k-d tree).  The
// host rasterises cell boxes with exactly this formula, and (x - lo) * inv is monotone in x, so q
// inside a box always maps to a cell inside the box's cell range.
__device__ __forceinline__ bool grid_cell(const Params& p, V q, uint32_t* cell) {
    const double fx = (q.x - p.grid_lo[0]) * p.grid_inv[0];
    const double fy = (q.y - p.grid_lo[1]) * p.grid_inv[1];
    const double fz = (q.z - p.grid_lo[2]) * p.grid_inv[2];
    if (!(fx >= 0.0 && fy >= 0.0 && fz >= 0.0 && fx < (double)p.grid_res[0] && fy < (double)p.grid_res[1] &&
          fz < (double)p.grid_res[2]))
        return false;
    *cell = ((uint32_t)fz * p.grid_res[1] + (uint32_t)fy) * p.grid_res[0] + (uint32_t)fx;
    return true;
}

}  // namespace dev
}  // namespace p2m
