// p2m_engine.cu -- the device engine behind the C ABI (include/p2m.h): packs the built structure
// into the device layout, uploads it to the first GPU, replicates it to the others by a one-time
// peer copy, and runs the query pipeline (Morton keys -> CUB radix sort -> fused query kernel).
//
// Multi-GPU: queries are independent (REF/SPEC.md:518-519), so p2m_query shards
// rows evenly over the engine's devices, one host thread per device, with no collective on the hot
// path; counters are summed on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <type_traits>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "../../../include/p2m.h"
#include "../host/geom.hpp"
#include "p2m_device.cuh"
#include "p2m_kernels.cuh"

#define P2M_API extern "C" __attribute__((visibility("default")))

extern "C" void p2m_set_last_error_internal(const char* msg);  // libp2m_host.so

using p2m::dev::D4;
using p2m::dev::Params;
using p2m::dev::kCy;

namespace {

void set_err(const std::string& s) { p2m_set_last_error_internal(s.c_str()); }

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) {                                                                 \
            set_err(std::string(#x) + ": " + cudaGetErrorString(e_));                            \
            return P2M_ERR_CUDA;                                                                 \
        }                                                                                        \
    } while (0)

// ---- host-side packing --------------------------------------------------------------------

constexpr uint64_t kListChunk = 256;  // = k_scan_tiles' chunk (p2m_grouped.cu kChunk)

// fn(s0, s1) over contiguous site ranges on all hardware threads
template <class Fn>
void parallel_sites(uint64_t S, Fn&& fn) {
    const unsigned T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const uint64_t step = std::max<uint64_t>(1024, (S + T * 8 - 1) / (T * 8));
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
        th.emplace_back([&] {
            for (;;) {
                const uint64_t a = next.fetch_add(step);
                if (a >= S) break;
                fn(a, std::min(S, a + step));
            }
        });
    for (auto& x : th) x.join();
}

float round_up_f(double v) {
    float f = (float)v;
    if ((double)f < v) f = std::nextafter(f, INFINITY);
    return f;
}

// Bounding cylinder of a set of faces for the scan's fp32 lower bound (p2m_grouped.cu cyl_near /
// the disk test): x = the faces' vertices (a face is the convex hull of its vertices and the cylinder
// is convex).  Axis n = the fp32 rounding of the unit area-weighted normal sum, centre c in fp32
// (cen if given -- a face's min-enclosing-sphere centre -- else the middle of the points' extents along
// n and two in-plane directions).  With nn = n / |n| in exact arithmetic, every point satisfies
// |nn.(x - c)| <= t and |x - c|^2 - (nn.(x - c))^2 <= R^2.  Stored {c, 4 R^2} and {n, t + tslack},
// both rounded up and inflated by 1e-12 (relative, and of the points' extent from c) over the fp64
// evaluation here (the device adds its fp32 error of |h| per row).
void fit_cyl(const double* x, int m, const double* nsum, const double* cen, float4* out) {
    double n[3] = {nsum[0], nsum[1], nsum[2]};
    double l = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    if (!(l > 0.0) || !std::isfinite(l)) { n[0] = 0.0; n[1] = 0.0; n[2] = 1.0; l = 1.0; }
    const float nf[3] = {(float)(n[0] / l), (float)(n[1] / l), (float)(n[2] / l)};
    const double lf = std::sqrt((double)nf[0] * nf[0] + (double)nf[1] * nf[1] + (double)nf[2] * nf[2]);
    const double nn[3] = {nf[0] / lf, nf[1] / lf, nf[2] / lf};
    double C[3];
    if (cen) {
        for (int k = 0; k < 3; ++k) C[k] = cen[k];
    } else {
        // in-plane basis e1, e2 perpendicular to nn
        double a[3] = {0.0, 0.0, 0.0};
        a[std::fabs(nn[0]) < 0.6 ? 0 : (std::fabs(nn[1]) < 0.6 ? 1 : 2)] = 1.0;
        double e1[3] = {a[1] * nn[2] - a[2] * nn[1], a[2] * nn[0] - a[0] * nn[2], a[0] * nn[1] - a[1] * nn[0]};
        const double l1 = std::sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
        for (double& v : e1) v /= l1;
        const double e2[3] = {nn[1] * e1[2] - nn[2] * e1[1], nn[2] * e1[0] - nn[0] * e1[2], nn[0] * e1[1] - nn[1] * e1[0]};
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int i = 0; i < m; ++i) {
            const double* p = x + 3 * i;
            const double c3[3] = {nn[0] * p[0] + nn[1] * p[1] + nn[2] * p[2], e1[0] * p[0] + e1[1] * p[1] + e1[2] * p[2],
                                  e2[0] * p[0] + e2[1] * p[1] + e2[2] * p[2]};
            for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], c3[k]); hi[k] = std::max(hi[k], c3[k]); }
        }
        const double mh = 0.5 * (lo[0] + hi[0]), m1 = 0.5 * (lo[1] + hi[1]), m2 = 0.5 * (lo[2] + hi[2]);
        for (int k = 0; k < 3; ++k) C[k] = nn[k] * mh + e1[k] * m1 + e2[k] * m2;
    }
    const float cf[3] = {(float)C[0], (float)C[1], (float)C[2]};
    double t = 0.0, r2 = 0.0, d2m = 0.0;
    for (int i = 0; i < m; ++i) {
        const double v[3] = {x[3 * i] - cf[0], x[3 * i + 1] - cf[1], x[3 * i + 2] - cf[2]};
        const double h = nn[0] * v[0] + nn[1] * v[1] + nn[2] * v[2];
        const double d2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
        t = std::max(t, std::fabs(h));
        r2 = std::max(r2, d2 - h * h);
        d2m = std::max(d2m, d2);
    }
    t = t * (1.0 + 1e-12) + 1e-12 * std::sqrt(d2m);
    r2 = r2 * (1.0 + 1e-12) + 1e-12 * d2m;
    out[0] = make_float4(cf[0], cf[1], cf[2], round_up_f(4.0 * r2));
    out[1] = make_float4(nf[0], nf[1], nf[2], round_up_f(t));
}

uint64_t lb_left_size(uint64_t n) {
    if (n <= 1) return 0;
    int d = 63 - __builtin_clzll(n);
    uint64_t full = (1ull << d) - 1ull, last = n - full, half = 1ull << (d - 1);
    return (half - 1ull) + std::min(last, half);
}

// Left-balanced k-d tree in BFS order: split on the widest axis of the subset's box (lowest axis on
// ties), the left subtree takes the lb_left_size(m) smallest points under (coordinate, site id).
// Same definition as the oracle's tree (oracle/p2m_oracle.c orc_kdtree_build).
void build_kdtree(const double* xyz, uint64_t n, std::vector<uint32_t>& node_site, std::vector<uint8_t>& node_dim) {
    node_site.assign(n, 0);
    node_dim.assign(n, 0);
    std::vector<uint32_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0u);
    struct T { uint64_t lo, hi, node; };
    std::vector<T> st;
    if (n) st.push_back({0, n, 0});
    while (!st.empty()) {
        T t = st.back();
        st.pop_back();
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (uint64_t i = t.lo; i < t.hi; ++i)
            for (int k = 0; k < 3; ++k) {
                double v = xyz[3 * (uint64_t)idx[i] + k];
                lo[k] = std::min(lo[k], v);
                hi[k] = std::max(hi[k], v);
            }
        int dim = 0;
        double ext = hi[0] - lo[0];
        if (hi[1] - lo[1] > ext) { dim = 1; ext = hi[1] - lo[1]; }
        if (hi[2] - lo[2] > ext) dim = 2;
        const uint64_t m = t.hi - t.lo, l = lb_left_size(m);
        std::nth_element(idx.begin() + t.lo, idx.begin() + t.lo + l, idx.begin() + t.hi, [&](uint32_t a, uint32_t b) {
            double ka = xyz[3 * (uint64_t)a + dim], kb = xyz[3 * (uint64_t)b + dim];
            return ka < kb || (ka == kb && a < b);
        });
        node_site[t.node] = idx[t.lo + l];
        node_dim[t.node] = (uint8_t)dim;
        if (t.hi > t.lo + l + 1) st.push_back({t.lo + l + 1, t.hi, 2 * t.node + 2});
        if (l > 0) st.push_back({t.lo, t.lo + l, 2 * t.node + 1});
    }
}

inline double bits_to_double(uint64_t b) { double d; std::memcpy(&d, &b, 8); return d; }

// Fallback BVH: median split of centroids on the longest centroid-box axis, leaf 4, DFS order.
struct FlatBvh {
    std::vector<D4> nodes;     // 2 per node
    std::vector<uint32_t> perm;
};

void build_bvh(const double* tri, uint64_t nf, FlatBvh& out) {
    out.nodes.clear();
    out.perm.resize(nf);
    std::iota(out.perm.begin(), out.perm.end(), 0u);
    if (!nf) return;
    std::vector<double> cen(3 * nf);
    for (uint64_t f = 0; f < nf; ++f)
        for (int k = 0; k < 3; ++k) cen[3 * f + k] = (tri[9 * f + k] + tri[9 * f + 3 + k] + tri[9 * f + 6 + k]) * (1.0 / 3.0);
    struct Rec {
        FlatBvh& o; const double* tri; const std::vector<double>& cen;
        uint32_t go(uint32_t lo, uint32_t hi) {
            uint32_t me = (uint32_t)(o.nodes.size() / 2);
            o.nodes.push_back(D4{}); o.nodes.push_back(D4{});
            double bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
            double cl[3] = {INFINITY, INFINITY, INFINITY}, ch[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (uint32_t i = lo; i < hi; ++i) {
                uint32_t f = o.perm[i];
                for (int v = 0; v < 3; ++v)
                    for (int k = 0; k < 3; ++k) {
                        double x = tri[9 * (uint64_t)f + 3 * v + k];
                        bl[k] = std::min(bl[k], x); bh[k] = std::max(bh[k], x);
                    }
                for (int k = 0; k < 3; ++k) { cl[k] = std::min(cl[k], cen[3 * (uint64_t)f + k]); ch[k] = std::max(ch[k], cen[3 * (uint64_t)f + k]); }
            }
            uint64_t meta;
            if (hi - lo <= 4) {
                meta = (uint64_t)(hi - lo) << 32 | lo;
            } else {
                int ax = 0;
                if (ch[1] - cl[1] > ch[ax] - cl[ax]) ax = 1;
                if (ch[2] - cl[2] > ch[ax] - cl[ax]) ax = 2;
                uint32_t mid = lo + (hi - lo) / 2;
                std::nth_element(o.perm.begin() + lo, o.perm.begin() + mid, o.perm.begin() + hi, [&](uint32_t a, uint32_t b) {
                    double x = cen[3 * (uint64_t)a + ax], y = cen[3 * (uint64_t)b + ax];
                    return x < y || (x == y && a < b);
                });
                go(lo, mid);
                uint32_t r = go(mid, hi);
                meta = r;
            }
            o.nodes[2 * me] = D4{bl[0], bl[1], bl[2], bh[0]};
            o.nodes[2 * me + 1] = D4{bh[1], bh[2], bits_to_double(meta), 0.0};
            return me;
        }
    } rec{out, tri, cen};
    rec.go(0, (uint32_t)nf);
}

// Host copy pool of the pageable-buffer path: a few persistent threads that split a list of memcpy
// segments into 2 MB pieces (one core's memcpy runs well below the host's memory bandwidth, and
// spawning threads per sub-chunk would cost more than the copy).  run() blocks; the caller works too.
class CopyPool {
  public:
    struct Seg { void* dst; const void* src; size_t bytes; };
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
    }
    ~CopyPool() {
        { std::lock_guard<std::mutex> lk(mu_); stop_ = true; }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void run(const Seg* segs, int nseg) {
        pieces_.clear();
        const size_t kPiece = 2u << 20;
        for (int i = 0; i < nseg; ++i)
            for (size_t o = 0; o < segs[i].bytes; o += kPiece)
                pieces_.push_back(Seg{(char*)segs[i].dst + o, (const char*)segs[i].src + o, std::min(kPiece, segs[i].bytes - o)});
        {
            std::lock_guard<std::mutex> lk(mu_);
            next_.store(0);
            busy_ = (int)th_.size();
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return busy_ == 0; });
    }
  private:
    void work() {
        for (size_t i; (i = next_.fetch_add(1)) < pieces_.size();) std::memcpy(pieces_[i].dst, pieces_[i].src, pieces_[i].bytes);
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
            std::lock_guard<std::mutex> lk(mu_);
            if (--busy_ == 0) done_.notify_all();
        }
    }
    std::vector<std::thread> th_;
    std::vector<Seg> pieces_;
    std::atomic<size_t> next_{0};
    std::mutex mu_;
    std::condition_variable cv_, done_;
    uint64_t gen_ = 0;
    int busy_ = 0;
    bool stop_ = false;
};

// Per-call working set of run_pipeline (keys/rows double buffers, CUB temp, tile arrays).
struct Scratch {
    uint32_t *keys = nullptr, *rows = nullptr, *keys2 = nullptr, *rows2 = nullptr;
    uint32_t *flag = nullptr, *tix = nullptr, *tiles = nullptr, *meta = nullptr, *tord = nullptr;
    void* tmp = nullptr;
    uint64_t n = 0, max_t = 0;
    size_t tb = 0;
};

void free_scratch(Scratch& c) {
    cudaFree(c.keys); cudaFree(c.rows); cudaFree(c.keys2); cudaFree(c.rows2); cudaFree(c.flag); cudaFree(c.tix);
    cudaFree(c.tiles); cudaFree(c.meta); cudaFree(c.tord); cudaFree(c.tmp);
    c = Scratch{};
}

struct Slot {
    int dev = 0;
    cudaStream_t stream = nullptr;
    D4 *kd = nullptr, *rec = nullptr, *bvh = nullptr;
    float4* fcy = nullptr;   // kCy float4 per face / batch / chunk: the bounding cylinders
    float4* bcy = nullptr;
    float4* ccy = nullptr;
    float4* bpt = nullptr;
    float4* cpt = nullptr;
    uint64_t* boff = nullptr;
    uint64_t* coff = nullptr;
    uint64_t* off = nullptr;
    uint32_t *lf = nullptr, *lfs = nullptr, *bvh_perm = nullptr;
    uint8_t* heavy = nullptr;
    D4* site_pos = nullptr;
    D4* site_ref = nullptr;
    uint32_t *grid_off = nullptr, *grid_site = nullptr;
    uint64_t* adj_off = nullptr;
    uint32_t* adj = nullptr;
    Params params{};
    std::mutex pmu;  // guards params (p2m_set_nns_strategy) against the snapshot every call takes
    std::mutex mu;
    // host-API path: kPipe streams, each with a chunk-sized staging set, so the H2D copy of one
    // chunk, the kernels of another and the D2H copy of a third overlap
    static constexpr int kPipe = 4;
    cudaStream_t pipe[kPipe] = {};
    cudaStream_t h2d = nullptr, d2h = nullptr;  // one in-order copy stream per PCIe direction
    // side streams of the small-tile scan, forked from / joined to the calling stream: [k] for the
    // host-API pipe k, [kPipe] for device-buffer calls
    cudaStream_t side[kPipe + 1] = {};
    cudaEvent_t fork[kPipe + 1] = {}, join[kPipe + 1] = {};
    std::mutex side_mu;  // device-buffer calls from several host threads share side[kPipe]: the
                         // fork/join event records and waits of one call must not interleave
    static constexpr int kMaxChunks = 64;
    std::vector<cudaEvent_t> cev;                // 3 per chunk: input landed, kernels done, output left
    cudaEvent_t t0 = nullptr;                    // P2M_E2E_TRACE origin
    struct Ws {
        double *q = nullptr, *dist = nullptr, *cp = nullptr;
        uint32_t *face = nullptr, *site = nullptr, *flags = nullptr;
        Scratch sc;  // the chunk's pipeline scratch: persistent, so chunks on different streams never
                     // wait on each other through the stream-ordered allocator's reuse dependencies
    } ws[kPipe];
    uint64_t cap = 0;   // rows per allocated staging set
    int nsets = 0;      // staging sets allocated (ws[0 .. nsets))
    // pageable host buffers (p2m_query): pinned bounce rings, sub-chunks of kRows rows.  The calling
    // thread packs input sub-chunks into the in-ring (host memcpy) and enqueues their H2D copies; a
    // second thread enqueues the D2H copies of finished chunks into the out-ring and unpacks them into
    // the caller's arrays, so both host copies overlap the kernels and the PCIe transfers.
    struct Bounce {
        static constexpr uint64_t kRows = 1ull << 20;
        static constexpr int kIn = 3, kOut = 4;
        double* in[kIn] = {};
        unsigned char* out[kOut] = {};   // dist 8 | cp 24 | face 4 | site 4 | flags 4 per row, as 5 arrays
        cudaEvent_t in_ev[kIn] = {}, out_ev[kOut] = {};
        std::unique_ptr<CopyPool> pack, unpack;  // host copy threads of the two directions
        bool ready = false;
    } bnc;
    cudaEvent_t agg_ready = nullptr;
    unsigned long long* agg = nullptr;
    // profiling: ring of event sets, read lazily by p2m_last_timings (no host sync per call)
    static constexpr int kRing = 256;
    static constexpr int kEv = 6;  // morton | sort | descend | regroup sort | scan | end
    std::vector<cudaEvent_t> ev;   // kEv per ring entry
    std::atomic<int> recorded{0};  // profiling-ring slots claimed (atomic: concurrent device calls)
};

}  // namespace

struct p2m_engine {
    std::vector<std::unique_ptr<Slot>> slots;
    double replicate_ms = 0.0;
    uint64_t bytes = 0;
    bool profiling = false;
    int scan_mode = P2M_SCAN_GROUPED;
    int morton_bits = -1;  // P2M_MORTON_BITS; auto: 24 up to 16 M rows (c2: one radix pass fewer, scan
                           // unchanged), 30 above (c5 at 100 M: the coarser order costs the scan more)
    int e2e_chunks = 0;
    double e2e_sched[4] = {1.0 / 32, 2.0, 0.25, 0.0};  // first, growth, cap, tail (P2M_E2E_SCHED)  // 0: geometric chunk schedule; k > 0: k equal chunks (P2M_E2E_CHUNKS, A/B)
    bool e2e_sched_set = false;  // P2M_E2E_SCHED given: no automatic choice between the dense and sparse schedules
    double e2e_sparse_tail = 0.1;  // sparse batches: one big chunk + a tail of this fraction (P2M_E2E_TAIL)
    uint64_t n_sites = 0, n_faces = 0, n_entries = 0, n_bvh = 0, n_heavy = 0;
    uint64_t grid_cells = 0, grid_pairs = 0;  // 0 = no grid (k-d tree only)
    uint64_t n_batches = 0;                   // 32-entry list batches (batch spheres)
    uint64_t n_chunks = 0;                    // 256-entry list chunks (chunk spheres)
    uint64_t n_adj = 0;                       // Delaunay adjacency entries (0 = no walk strategy)
    bool has_adj = false;
};

namespace {

void free_slot(Slot& s) {
    cudaSetDevice(s.dev);
    cudaFree(s.kd); cudaFree(s.rec); cudaFree(s.bvh); cudaFree(s.off); cudaFree(s.lf); cudaFree(s.bvh_perm);
    cudaFree(s.heavy);
    cudaFree(s.site_pos); cudaFree(s.site_ref); cudaFree(s.grid_off); cudaFree(s.grid_site);
    cudaFree(s.fcy); cudaFree(s.bcy); cudaFree(s.ccy);
    cudaFree(s.bpt); cudaFree(s.boff);
    cudaFree(s.cpt); cudaFree(s.coff); cudaFree(s.lfs);
    cudaFree(s.adj_off); cudaFree(s.adj);
    for (auto& w : s.ws) {
        cudaFree(w.q); cudaFree(w.dist); cudaFree(w.cp); cudaFree(w.face); cudaFree(w.site); cudaFree(w.flags);
        free_scratch(w.sc);
    }
    for (auto& st : s.pipe) if (st) cudaStreamDestroy(st);
    if (s.h2d) cudaStreamDestroy(s.h2d);
    for (int k = 0; k <= Slot::kPipe; ++k) {
        if (s.side[k]) cudaStreamDestroy(s.side[k]);
        if (s.fork[k]) cudaEventDestroy(s.fork[k]);
        if (s.join[k]) cudaEventDestroy(s.join[k]);
    }
    if (s.d2h) cudaStreamDestroy(s.d2h);
    for (auto& e : s.cev) if (e) cudaEventDestroy(e);
    s.cev.clear();
    if (s.t0) cudaEventDestroy(s.t0);
    if (s.agg_ready) cudaEventDestroy(s.agg_ready);
    for (auto& b : s.bnc.in) if (b) cudaFreeHost(b);
    for (auto& b : s.bnc.out) if (b) cudaFreeHost(b);
    for (auto& e : s.bnc.in_ev) if (e) cudaEventDestroy(e);
    for (auto& e : s.bnc.out_ev) if (e) cudaEventDestroy(e);
    cudaFree(s.agg);
    for (auto& e : s.ev) if (e) cudaEventDestroy(e);
    s.ev.clear();
    if (s.stream) cudaStreamDestroy(s.stream);
}

// Exact cell-locate grid over the Morton key box (1.5x the real sites' AABB): cubic cells, about 16
// per real site, at most 512 per axis; site s is listed in every cell its Voronoi cell box (inflated
// by 1e-9 |D|) meets.  Built only when (1) every real site has a box and (2) no sentinel can be
// nearest anywhere in the grid box: with s0 the real site nearest the box centre, every point x of
// the box has d(x, nearest real) <= max_corner |corner - s0| < min_k d(sentinel_k, box).
struct Grid {
    double lo[3] = {0, 0, 0}, inv[3] = {0, 0, 0};
    uint32_t res[3] = {0, 0, 0};
    std::vector<uint32_t> off, site;
};

}  // namespace
namespace p2m { namespace dev {
bool build_grid_device(int dev, const D4* kd_host, uint32_t S, const double lo[3], const double inv[3],
                       const uint32_t res[3], std::vector<uint32_t>& off, std::vector<uint32_t>& site);
} }
namespace {

// Without cell boxes (an external builder's desc) the same grid is built on device `dev` from the
// sites alone (p2m_grid.cu: k-d radius search + the affine bisector test at the cell corners).
bool build_grid(const p2m_engine_desc* d, const double* key_lo, const double* key_ext, Grid& g,
                const std::vector<D4>& kd, int dev) {
    const uint64_t S = d->n_sites;
    double hi[3], c[3];
    for (int k = 0; k < 3; ++k) { hi[k] = key_lo[k] + key_ext[k]; c[k] = 0.5 * (key_lo[k] + hi[k]); }
    uint64_t n_real = 0, s0 = UINT64_MAX;
    double best = INFINITY;
    for (uint64_t s = 0; s < S; ++s) {
        if (d->site_kind[s] == P2M_SITE_SENTINEL) continue;
        ++n_real;
        if (d->site_cell_box) {
            const double* b = d->site_cell_box + 6 * s;
            for (int k = 0; k < 6; ++k) if (!std::isfinite(b[k])) return false;
        }
        const double* p = d->site_xyz + 3 * s;
        const double dd = (p[0] - c[0]) * (p[0] - c[0]) + (p[1] - c[1]) * (p[1] - c[1]) + (p[2] - c[2]) * (p[2] - c[2]);
        if (dd < best) { best = dd; s0 = s; }
    }
    if (!n_real) return false;
    double rmax = 0.0;
    for (int i = 0; i < 8; ++i) {
        double dd = 0.0;
        for (int k = 0; k < 3; ++k) {
            const double x = (i >> k & 1) ? hi[k] : key_lo[k];
            dd += (x - d->site_xyz[3 * s0 + k]) * (x - d->site_xyz[3 * s0 + k]);
        }
        rmax = std::max(rmax, std::sqrt(dd));
    }
    for (uint64_t s = 0; s < S; ++s) {
        if (d->site_kind[s] != P2M_SITE_SENTINEL) continue;
        double dd = 0.0;
        for (int k = 0; k < 3; ++k) {
            const double x = d->site_xyz[3 * s + k];
            const double t = x < key_lo[k] ? key_lo[k] - x : (x > hi[k] ? x - hi[k] : 0.0);
            dd += t * t;
        }
        if (!(std::sqrt(dd) > rmax * (1.0 + 1e-9))) return false;
    }
    const double vol = key_ext[0] * key_ext[1] * key_ext[2];
    const double cell = std::cbrt(vol / (16.0 * (double)n_real));
    for (int k = 0; k < 3; ++k) {
        g.lo[k] = key_lo[k];
        g.res[k] = (uint32_t)std::min(512.0, std::max(1.0, std::ceil(key_ext[k] / cell)));
        g.inv[k] = (double)g.res[k] / key_ext[k];
    }
    if (!d->site_cell_box) {
        if (std::getenv("P2M_NO_DEVICE_GRID")) return false;
        return p2m::dev::build_grid_device(dev, kd.data(), (uint32_t)S, g.lo, g.inv, g.res, g.off, g.site);
    }
    double dspan = 0.0;
    for (int k = 0; k < 3; ++k) dspan += (d->domain_max[k] - d->domain_min[k]) * (d->domain_max[k] - d->domain_min[k]);
    const double margin = 1e-9 * std::sqrt(dspan);
    const uint64_t ncell = (uint64_t)g.res[0] * g.res[1] * g.res[2];
    auto range = [&](const double* b, uint32_t* i0, uint32_t* i1) {
        for (int k = 0; k < 3; ++k) {
            const double a = (b[k] - margin - g.lo[k]) * g.inv[k], z = (b[3 + k] + margin - g.lo[k]) * g.inv[k];
            if (z < 0.0 || a >= (double)g.res[k]) return false;
            i0[k] = a <= 0.0 ? 0u : (uint32_t)std::min<double>(std::floor(a), g.res[k] - 1);
            i1[k] = z <= 0.0 ? 0u : (uint32_t)std::min<double>(std::floor(z), g.res[k] - 1);
        }
        return true;
    };
    std::vector<uint64_t> cnt(ncell + 1, 0);
    uint32_t i0[3], i1[3];
    for (int pass = 0; pass < 2; ++pass) {
        std::vector<uint64_t> cur;
        if (pass == 1) {
            for (uint64_t cidx = 0; cidx < ncell; ++cidx) cnt[cidx + 1] += cnt[cidx];
            if (cnt[ncell] >= (1ull << 32)) return false;
            g.site.resize(cnt[ncell]);
            cur.assign(cnt.begin(), cnt.end() - 1);
        }
        for (uint64_t s = 0; s < S; ++s) {
            if (d->site_kind[s] == P2M_SITE_SENTINEL) continue;
            if (!range(d->site_cell_box + 6 * s, i0, i1)) continue;
            for (uint32_t z = i0[2]; z <= i1[2]; ++z)
                for (uint32_t y = i0[1]; y <= i1[1]; ++y)
                    for (uint32_t x = i0[0]; x <= i1[0]; ++x) {
                        const uint64_t cidx = ((uint64_t)z * g.res[1] + y) * g.res[0] + x;
                        if (pass == 0) ++cnt[cidx + 1];
                        else g.site[cur[cidx]++] = (uint32_t)s;
                    }
        }
    }
    g.off.resize(ncell + 1);
    for (uint64_t cidx = 0; cidx <= ncell; ++cidx) g.off[cidx] = (uint32_t)cnt[cidx];
    return true;
}

int alloc_slot(Slot& s, const p2m_engine& E) {
    CK(cudaSetDevice(s.dev));
    CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    for (auto& st : s.pipe) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s.h2d, cudaStreamNonBlocking));
    for (int k = 0; k <= Slot::kPipe; ++k) {
        CK(cudaStreamCreateWithFlags(&s.side[k], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&s.fork[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&s.join[k], cudaEventDisableTiming));
    }
    CK(cudaStreamCreateWithFlags(&s.d2h, cudaStreamNonBlocking));
    s.cev.assign(3 * Slot::kMaxChunks, nullptr);
    // timing-capable only under P2M_E2E_TRACE (per-chunk timeline on stderr)
    const bool trace = std::getenv("P2M_E2E_TRACE") != nullptr;
    for (auto& e : s.cev) CK(cudaEventCreateWithFlags(&e, trace ? cudaEventDefault : cudaEventDisableTiming));
    if (trace) CK(cudaEventCreate(&s.t0));
    CK(cudaEventCreateWithFlags(&s.agg_ready, cudaEventDisableTiming));
    CK(cudaMalloc(&s.kd, sizeof(D4) * std::max<uint64_t>(1, E.n_sites)));
    CK(cudaMalloc(&s.rec, sizeof(D4) * 4 * std::max<uint64_t>(1, E.n_faces)));
    CK(cudaMalloc(&s.fcy, sizeof(float4) * kCy * std::max<uint64_t>(1, E.n_faces)));
    CK(cudaMalloc(&s.bcy, sizeof(float4) * kCy * std::max<uint64_t>(1, E.n_batches)));
    CK(cudaMalloc(&s.ccy, sizeof(float4) * kCy * std::max<uint64_t>(1, E.n_chunks)));
    CK(cudaMalloc(&s.bpt, sizeof(float4) * std::max<uint64_t>(1, E.n_batches)));
    CK(cudaMalloc(&s.boff, sizeof(uint64_t) * (E.n_sites + 1)));
    CK(cudaMalloc(&s.off, sizeof(uint64_t) * (E.n_sites + 1)));
    CK(cudaMalloc(&s.lf, sizeof(uint32_t) * std::max<uint64_t>(1, E.n_entries)));
    CK(cudaMalloc(&s.lfs, sizeof(uint32_t) * std::max<uint64_t>(1, E.n_entries)));
    CK(cudaMalloc(&s.cpt, sizeof(float4) * std::max<uint64_t>(1, E.n_chunks)));
    CK(cudaMalloc(&s.coff, sizeof(uint64_t) * (E.n_sites + 1)));
    CK(cudaMalloc(&s.bvh, sizeof(D4) * 2 * std::max<uint64_t>(1, E.n_bvh)));
    CK(cudaMalloc(&s.bvh_perm, sizeof(uint32_t) * std::max<uint64_t>(1, E.n_faces)));
    CK(cudaMalloc(&s.agg, sizeof(unsigned long long) * 8));
    CK(cudaMalloc(&s.heavy, std::max<uint64_t>(1, E.n_sites)));
    CK(cudaMalloc(&s.site_pos, sizeof(D4) * std::max<uint64_t>(1, E.n_sites)));
    CK(cudaMalloc(&s.site_ref, sizeof(D4) * std::max<uint64_t>(1, E.n_sites)));
    if (E.has_adj) {
        CK(cudaMalloc(&s.adj_off, 8 * (E.n_sites + 1)));
        CK(cudaMalloc(&s.adj, 4 * std::max<uint64_t>(1, E.n_adj)));
    }
    if (E.grid_cells) {
        CK(cudaMalloc(&s.grid_off, 4 * (E.grid_cells + 1)));
        CK(cudaMalloc(&s.grid_site, 4 * std::max<uint64_t>(1, E.grid_pairs)));
    }
    CK(cudaMemset(s.heavy, 0, std::max<uint64_t>(1, E.n_sites)));
    s.ev.assign(Slot::kEv * Slot::kRing, nullptr);
    for (auto& e : s.ev) CK(cudaEventCreate(&e));
    // keep the stream-ordered pool's memory between calls (the per-call sort workspace)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, s.dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return P2M_OK;
}

int ensure_scratch(Scratch& c, uint64_t n, uint64_t n_sites);

// Staging sets 0 .. nsets-1 of the host-API pipeline, each for chunks of up to n rows (a schedule of
// c chunks only ever uses min(c, kPipe) sets: two big chunks must not pay for four).
int ensure_ws(Slot& s, uint64_t n, uint64_t n_sites, int nsets) {
    nsets = std::min(std::max(nsets, 1), (int)Slot::kPipe);
    if (n <= s.cap && nsets <= s.nsets) return P2M_OK;
    CK(cudaDeviceSynchronize());
    n = std::max(n, s.cap);
    nsets = std::max(nsets, s.nsets);
    s.cap = 0;
    s.nsets = 0;
    for (int k = 0; k < Slot::kPipe; ++k) {
        auto& w = s.ws[k];
        cudaFree(w.q); cudaFree(w.dist); cudaFree(w.cp); cudaFree(w.face); cudaFree(w.site); cudaFree(w.flags);
        free_scratch(w.sc);
        w = Slot::Ws{};
        if (k >= nsets) continue;
        CK(cudaMalloc(&w.q, 24 * n));
        CK(cudaMalloc(&w.dist, 8 * n));
        CK(cudaMalloc(&w.cp, 24 * n));
        CK(cudaMalloc(&w.face, 4 * n));
        CK(cudaMalloc(&w.site, 4 * n));
        CK(cudaMalloc(&w.flags, 4 * n));
        int rc = ensure_scratch(w.sc, n, n_sites);
        if (rc != P2M_OK) return rc;
    }
    s.cap = n;
    s.nsets = nsets;
    return P2M_OK;
}

size_t pipeline_tmp_bytes(uint64_t n, uint64_t max_t, bool lpt) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int64_t)n, 0, 30, (cudaStream_t)0);
    tb = std::max(tb, p2m::dev::tiles_tmp_bytes(n));
    if (lpt) tb = std::max(tb, p2m::dev::tile_order_tmp_bytes(max_t));
    return tb;
}

// Persistent scratch for calls of up to n rows (synchronous allocation: call before a pipeline).
int ensure_scratch(Scratch& c, uint64_t n, uint64_t n_sites) {
    if (n <= c.n) return P2M_OK;
    free_scratch(c);
    const uint64_t max_t = p2m::dev::max_tiles(n, n_sites);
    c.tb = pipeline_tmp_bytes(n, max_t, true);
    CK(cudaMalloc(&c.keys, 4 * n)); CK(cudaMalloc(&c.rows, 4 * n));
    CK(cudaMalloc(&c.keys2, 4 * n)); CK(cudaMalloc(&c.rows2, 4 * n));
    CK(cudaMalloc(&c.flag, 4 * n)); CK(cudaMalloc(&c.tix, 4 * n));
    CK(cudaMalloc(&c.tiles, 4 * max_t)); CK(cudaMalloc(&c.meta, 16)); CK(cudaMalloc(&c.tord, 16 * max_t));
    CK(cudaMalloc(&c.tmp, c.tb));
    c.n = n;
    c.max_t = max_t;
    return P2M_OK;
}

// Morton keys -> sort -> descend -> regroup -> tile scan (or the fused per-row query).  sc: a
// persistent scratch of >= n rows, else the working set comes from the stream-ordered allocator.
int run_pipeline(p2m_engine* E, Slot& s, const double* d_q, uint64_t n, const p2m::dev::Out& o, bool counters,
                 cudaStream_t st, bool nearest_only, uint32_t* d_site_only, bool allow_prof = true,
                 Scratch* sc = nullptr, int side = Slot::kPipe) {
    if (n >= (1ull << 32)) { set_err("p2m_query_device: at most 2^32-1 rows per call"); return P2M_ERR_INVALID; }
    CK(cudaSetDevice(s.dev));
    uint32_t *keys = nullptr, *rows = nullptr, *keys2 = nullptr, *rows2 = nullptr;
    void* tmp = nullptr;
    uint32_t *flag = nullptr, *tix = nullptr, *tiles = nullptr, *meta = nullptr;
    const bool grouped = !nearest_only && E->scan_mode == P2M_SCAN_GROUPED;
    const uint64_t max_t = p2m::dev::max_tiles(n, E->n_sites);
    // launch order of the scan tiles (P2M_TILE_ORDER): measured on c2, longest-first wins below a
    // few million rows (the heaviest tiles otherwise start last and set the tail) and site order
    // above (neighbouring tiles share lists in L2); -1 = choose by batch size
    Params sp;
    {
        std::lock_guard<std::mutex> lk(s.pmu);
        sp = s.params;  // one consistent snapshot per call
    }
    // warp tiles for the sites that are not heavy when rows are sparse per site (measured: c5, 51 rows
    // per site, +2%, c1 +13%; dense batches -- c2, 570 rows per site -- keep the CTA tiles, whose
    // staged chunks serve up to 256 rows); P2M_WARP_MIN_CHUNKS overrides (0 = off)
    if (sp.warp_min_chunks == ~0u) sp.warp_min_chunks = (n < 128ull * E->n_sites) ? 1u : 0u;
    int order = sp.tile_order;
    if (order < 0) order = n < (4ull << 20) ? 1 : 0;
    const bool lpt = true;  // the launch order array (site order, LPT or buckets; small tiles last) always exists
    uint32_t* tord = nullptr;  // 4 x max_t: keys, sorted keys, tile ids, launch order
    size_t tb = 0;
    const bool own = sc == nullptr || sc->n < n;
    if (!own) {
        keys = sc->keys; rows = sc->rows; keys2 = sc->keys2; rows2 = sc->rows2; tmp = sc->tmp; tb = sc->tb;
        flag = sc->flag; tix = sc->tix; tiles = sc->tiles; meta = sc->meta;
        if (grouped && lpt) tord = sc->tord;
    } else {
        tb = pipeline_tmp_bytes(n, max_t, grouped && lpt);
        CK(cudaMallocAsync(&keys, 4 * n, st));
        CK(cudaMallocAsync(&rows, 4 * n, st));
        CK(cudaMallocAsync(&keys2, 4 * n, st));
        CK(cudaMallocAsync(&rows2, 4 * n, st));
        CK(cudaMallocAsync(&tmp, tb, st));
        if (grouped) {
            CK(cudaMallocAsync(&flag, 4 * n, st));
            CK(cudaMallocAsync(&tix, 4 * n, st));
            CK(cudaMallocAsync(&tiles, 4 * max_t, st));
            CK(cudaMallocAsync(&meta, 16, st));
            if (lpt) CK(cudaMallocAsync(&tord, 16 * max_t, st));
        }
    }
    int ring = -1;
    if (allow_prof && E->profiling && s.recorded.load() < Slot::kRing) {
        ring = s.recorded.fetch_add(1);
        if (ring >= Slot::kRing) ring = -1;
    }
    const bool prof = ring >= 0;
    cudaEvent_t* ev = prof ? &s.ev[Slot::kEv * ring] : nullptr;
    if (prof) CK(cudaEventRecord(ev[0], st));
    CK(p2m::dev::launch_morton(d_q, n, sp, keys, rows, st));
    if (prof) CK(cudaEventRecord(ev[1], st));
    // the Morton order only has to be spatially coherent: sorting on the top morton_bits of the
    // 30-bit key saves radix passes (8 bits per onesweep pass)
    const int mbits = E->morton_bits > 0 ? E->morton_bits : (n > (16ull << 20) ? 30 : 24);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, rows, rows2, (int64_t)n, 30 - mbits, 30, st));
    if (prof) CK(cudaEventRecord(ev[2], st));
    if (nearest_only) {
        CK(p2m::dev::launch_nearest(sp, d_q, rows2, n, d_site_only, st));
        if (prof) for (int k = 3; k < Slot::kEv; ++k) CK(cudaEventRecord(ev[k], st));
    } else if (E->scan_mode == P2M_SCAN_FUSED) {
        CK(p2m::dev::launch_query(sp, d_q, rows2, n, o, counters, st));
        if (prof) for (int k = 3; k < Slot::kEv; ++k) CK(cudaEventRecord(ev[k], st));
    } else {
        // descend in Morton order (keys buffer reused for the site keys), regroup by site (stable),
        // then scan per site tile
        CK(p2m::dev::launch_descend(sp, d_q, rows2, n, keys, o, counters, st));
        if (prof) CK(cudaEventRecord(ev[3], st));
        const int bits = std::max(1, 64 - __builtin_clzll((unsigned long long)E->n_sites));  // keys <= n_sites
        CK(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, rows2, rows, (int64_t)n, 0, bits, st));
        // tiles over the site-sorted order (keys / rows2 are free again: hpos / run starts)
        CK(p2m::dev::launch_tiles(sp, keys2, n, (uint32_t)E->n_sites, keys, rows2, flag, tix, tiles, meta, tmp, tb, st));
        if (prof) CK(cudaEventRecord(ev[4], st));
        const char* trace_path = std::getenv("P2M_TILE_TRACE");
        unsigned long long* trace = nullptr;
        const uint64_t ntile_max = p2m::dev::max_tiles(n, E->n_sites);
        Params prm = sp;
        prm.tile_order = order;
        if (trace_path) {  // debug: per-tile timing dump (scripts/tile_trace.py)
            CK(cudaMallocAsync(&trace, 32 * ntile_max, st));
            CK(cudaMemsetAsync(trace, 0, 32 * ntile_max, st));
            prm.tile_trace = trace;
        }
        if (tord)
            CK(p2m::dev::launch_tile_order(prm, keys2, tiles, meta, max_t, tord, tord + max_t, tord + 2 * max_t,
                                           tord + 3 * max_t, tmp, tb, st));
        {
            std::unique_lock<std::mutex> lk(s.side_mu, std::defer_lock);
            if (side == Slot::kPipe) lk.lock();  // host-API pipes run under the slot mutex already
            p2m::dev::Out om = o;
            om.miss = tix;                       // free after tile construction: the table-miss queue
            om.miss_n = meta + 3;
            CK(p2m::dev::launch_scan_tiles(prm, d_q, rows, keys2, tiles, meta, tord ? tord + 3 * max_t : nullptr, n,
                                           om, counters, st, s.side[side], s.fork[side], s.join[side]));
            CK(p2m::dev::launch_table_miss(prm, d_q, om, st));
        }
        if (trace) {
            std::vector<unsigned long long> h(4 * ntile_max);
            CK(cudaMemcpyAsync(h.data(), trace, 32 * ntile_max, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (FILE* fp = std::fopen(trace_path, "wb")) { std::fwrite(h.data(), 8, h.size(), fp); std::fclose(fp); }
            CK(cudaFreeAsync(trace, st));
        }
        if (prof) CK(cudaEventRecord(ev[5], st));
    }
    if (!own) return P2M_OK;
    CK(cudaFreeAsync(keys, st));
    CK(cudaFreeAsync(rows, st));
    CK(cudaFreeAsync(keys2, st));
    CK(cudaFreeAsync(rows2, st));
    CK(cudaFreeAsync(tmp, st));
    if (grouped) {
        CK(cudaFreeAsync(flag, st));
        CK(cudaFreeAsync(tix, st));
        CK(cudaFreeAsync(tiles, st));
        CK(cudaFreeAsync(meta, st));
        if (tord) CK(cudaFreeAsync(tord, st));
    }
    return P2M_OK;
}

// Per-site exact-work estimate: query every site's own position once with the sequential (fused)
// scan and count the exact point-triangle evaluations.  Sites whose estimate reaches the threshold
// (deep auxiliary sites of closed surfaces, where the distance field is flat and sphere pruning
// cannot cut the list) get short tiles so their rows spread over many SMs.
int mark_heavy_sites(p2m_engine* E, const double* site_xyz, const uint8_t* site_kind) {
    uint32_t thr = 1024;
    if (const char* v = std::getenv("P2M_HEAVY_E")) thr = (uint32_t)std::strtoul(v, nullptr, 10);
    const uint64_t S = E->n_sites;
    Slot& s0 = *E->slots[0];
    CK(cudaSetDevice(s0.dev));
    double *q = nullptr, *dist = nullptr, *cp = nullptr;
    uint32_t *face = nullptr, *site = nullptr;
    uint64_t* pq = nullptr;
    CK(cudaMalloc(&q, 24 * S)); CK(cudaMalloc(&dist, 8 * S)); CK(cudaMalloc(&cp, 24 * S));
    CK(cudaMalloc(&face, 4 * S)); CK(cudaMalloc(&site, 4 * S)); CK(cudaMalloc(&pq, 24 * S));
    CK(cudaMemcpy(q, site_xyz, 24 * S, cudaMemcpyHostToDevice));
    const int mode = E->scan_mode;
    const bool prof = E->profiling;
    E->scan_mode = P2M_SCAN_FUSED;
    E->profiling = false;
    p2m::dev::Out o{dist, cp, face, site, nullptr, pq, nullptr};
    int rc = run_pipeline(E, s0, q, S, o, true, s0.stream, false, nullptr);
    E->scan_mode = mode;
    E->profiling = prof;
    std::vector<uint64_t> h(3 * S);
    if (rc == P2M_OK) {
        CK(cudaStreamSynchronize(s0.stream));
        CK(cudaMemcpy(h.data(), pq, 24 * S, cudaMemcpyDeviceToHost));
    }
    cudaFree(q); cudaFree(dist); cudaFree(cp); cudaFree(face); cudaFree(site); cudaFree(pq);
    if (rc != P2M_OK) return rc;
    std::vector<uint8_t> heavy(S, 0);
    uint64_t n_heavy = 0;
    for (uint64_t i = 0; i < S; ++i)
        if (site_kind[i] != P2M_SITE_SENTINEL && h[3 * i + 1] >= thr) { heavy[i] = 1; ++n_heavy; }
    E->n_heavy = n_heavy;
    for (auto& s : E->slots) {
        CK(cudaSetDevice(s->dev));
        CK(cudaMemcpy(s->heavy, heavy.data(), S, cudaMemcpyHostToDevice));
    }
    return P2M_OK;
}


// The packed device layout of one replica as host arrays: what p2m_engine_create derives from a
// p2m_engine_desc, and what a device image file (p2m_engine_save / p2m_engine_load) stores.
struct Image {
    template <class T>
    struct Arr {
        const T* p = nullptr;
        uint64_t n = 0;
        std::vector<T> own;
        void set(const T* q, uint64_t m) { p = q; n = m; }
        void take(std::vector<T>&& v) { own = std::move(v); p = own.data(); n = own.size(); }
        uint64_t bytes() const { return sizeof(T) * n; }
    };
    Arr<D4> kd, rec, bvh, site_pos, site_ref;
    Arr<float4> fcy, bcy, ccy, bpt, cpt;
    Arr<uint64_t> boff, coff, off, adj_off;
    Arr<uint32_t> lf, lfs, bvh_perm, grid_off, grid_site, adj;
    Arr<uint8_t> heavy;   // empty: estimate at creation (mark_heavy_sites)
};

// Allocate the slots, upload the image to the first device, replicate it to the others by a one-time
// peer copy, set the kernel parameters and the schedule knobs; E's counts must be set.
int upload_engine(p2m_engine* E, const Params& P, const Image& I, int n_devices, const int* device_ids, int ndev) {
    const uint64_t S = E->n_sites, F = E->n_faces;
    for (int k = 0; k < n_devices; ++k) {
        auto s = std::make_unique<Slot>();
        s->dev = device_ids ? device_ids[k] : k;
        if (s->dev < 0 || s->dev >= ndev) { set_err("p2m_engine_create: bad device id"); return P2M_ERR_INVALID; }
        E->slots.push_back(std::move(s));
    }
    for (auto& s : E->slots) {
        int rc = alloc_slot(*s, *E);
        if (rc != P2M_OK) return rc;
    }
    Slot& s0 = *E->slots[0];
    struct Up { void* dst; const void* src; size_t n; };
    auto uploads = [&](Slot& s) {
        return std::vector<Up>{
            {s.kd, I.kd.p, I.kd.bytes()}, {s.rec, I.rec.p, I.rec.bytes()}, {s.fcy, I.fcy.p, I.fcy.bytes()},
            {s.bcy, I.bcy.p, I.bcy.bytes()}, {s.ccy, I.ccy.p, I.ccy.bytes()},
            {s.bpt, I.bpt.p, I.bpt.bytes()}, {s.boff, I.boff.p, I.boff.bytes()},
            {s.off, I.off.p, I.off.bytes()}, {s.lf, I.lf.p, I.lf.bytes()}, {s.lfs, I.lfs.p, I.lfs.bytes()},
            {s.cpt, I.cpt.p, I.cpt.bytes()}, {s.coff, I.coff.p, I.coff.bytes()}, {s.bvh, I.bvh.p, I.bvh.bytes()},
            {s.bvh_perm, I.bvh_perm.p, I.bvh_perm.bytes()}, {s.site_pos, I.site_pos.p, I.site_pos.bytes()},
            {s.site_ref, I.site_ref.p, I.site_ref.bytes()},
            {s.adj_off, I.adj_off.p, E->has_adj ? I.adj_off.bytes() : 0}, {s.adj, I.adj.p, E->has_adj ? I.adj.bytes() : 0},
            {s.grid_off, I.grid_off.p, E->grid_cells ? I.grid_off.bytes() : 0},
            {s.grid_site, I.grid_site.p, E->grid_cells ? I.grid_site.bytes() : 0},
            {s.heavy, I.heavy.p, I.heavy.bytes()}};
    };
    {
        CK(cudaSetDevice(s0.dev));
        for (const Up& u : uploads(s0))
            if (u.n && cudaMemcpy(u.dst, u.src, u.n, cudaMemcpyHostToDevice) != cudaSuccess) {
                set_err(std::string("p2m_engine_create: upload failed: ") + cudaGetErrorString(cudaGetLastError()));
                return P2M_ERR_CUDA;
            }
    }
    E->bytes = 0;
    for (const Up& u : uploads(s0)) E->bytes += u.n;
    auto t0 = std::chrono::steady_clock::now();
    for (size_t k = 1; k < E->slots.size(); ++k) {
        Slot& s = *E->slots[k];
        cudaSetDevice(s.dev);
        if (s.dev != s0.dev) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, s.dev, s0.dev);
            if (can) {
                cudaError_t e = cudaDeviceEnablePeerAccess(s0.dev, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) { set_err("peer access failed"); return P2M_ERR_CUDA; }
                cudaGetLastError();
            }
        }
        const std::vector<Up> dst = uploads(s), src = uploads(s0);
        for (size_t i = 0; i < dst.size(); ++i)
            if (dst[i].n && cudaMemcpyPeerAsync(dst[i].dst, s.dev, src[i].dst, s0.dev, dst[i].n, s.stream) != cudaSuccess) {
                set_err("p2m_engine_create: peer copy failed");
                return P2M_ERR_CUDA;
            }
    }
    for (auto& s : E->slots) {
        cudaSetDevice(s->dev);
        if (cudaStreamSynchronize(s->stream) != cudaSuccess) { set_err("p2m_engine_create: replica sync failed"); return P2M_ERR_CUDA; }
    }
    E->replicate_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (auto& s : E->slots) {
        s->params = P;
        s->params.kd = s->kd; s->params.rec = s->rec; s->params.fcy = s->fcy; s->params.bcy = s->bcy; s->params.ccy = s->ccy; s->params.bpt = s->bpt; s->params.boff = s->boff; s->params.off = s->off; s->params.lf = s->lf;
        s->params.lfs = s->lfs; s->params.cpt = s->cpt; s->params.coff = s->coff;
        s->params.bvh = s->bvh; s->params.bvh_perm = s->bvh_perm; s->params.heavy = s->heavy;
        s->params.site_pos = s->site_pos;
        s->params.site_ref = s->site_ref;
        s->params.grid_off = E->grid_cells ? s->grid_off : nullptr;
        s->params.grid_site = s->grid_site;
        s->params.nns = P2M_NNS_GRID;
        s->params.tile_order = -1;
        s->params.small_chunks = 2;  // measured on c2 (1, 2 > 4) and c5 (2 ~ 4 > 0)
        if (const char* v = std::getenv("P2M_SMALL_CHUNKS")) s->params.small_chunks = (uint32_t)std::min(4, std::max(0, std::atoi(v)));
        if (const char* v = std::getenv("P2M_TILE_ORDER")) s->params.tile_order = std::atoi(v);
        s->params.warp_tiles = 0;
        if (const char* v = std::getenv("P2M_SCAN_WARP")) s->params.warp_tiles = std::atoi(v) ? 1 : 0;
        s->params.warp_queue = std::getenv("P2M_NO_WARP_QUEUE") ? 0 : 1;
        s->params.tvote = std::getenv("P2M_NO_TVOTE") ? 0 : 1;
        s->params.dense_pairs = 12u;
        if (const char* v = std::getenv("P2M_DENSE_PAIRS")) s->params.dense_pairs = (uint32_t)std::max(1, std::atoi(v));
        s->params.warp_min_chunks = ~0u;  // auto (run_pipeline)
        if (const char* v = std::getenv("P2M_WARP_MIN_CHUNKS")) s->params.warp_min_chunks = (uint32_t)std::max(0, std::atoi(v));
        s->params.adj_off = E->has_adj ? s->adj_off : nullptr;
        s->params.adj = s->adj;
    }
    if (const char* v = std::getenv("P2M_MORTON_BITS")) E->morton_bits = std::min(30, std::max(3, std::atoi(v)));
    if (const char* v = std::getenv("P2M_E2E_SCHED")) {
        double x[4];
        if (std::sscanf(v, "%lf,%lf,%lf,%lf", &x[0], &x[1], &x[2], &x[3]) == 4 && x[0] > 0 && x[1] >= 1 && x[2] > 0 &&
            x[3] >= 0 && x[3] < 1)
        {
            for (int k = 0; k < 4; ++k) E->e2e_sched[k] = x[k];
            E->e2e_sched_set = true;
        }
    }
    if (const char* v = std::getenv("P2M_E2E_TAIL")) {
        const double t = std::atof(v);
        if (t >= 0 && t < 1) E->e2e_sparse_tail = t;
    }
    if (const char* v = std::getenv("P2M_E2E_CHUNKS")) E->e2e_chunks = std::max(0, std::atoi(v));
    return P2M_OK;
}

}  // namespace

// =============================================================================================

P2M_API int p2m_engine_create(const p2m_engine_desc* d, int n_devices, const int* device_ids, p2m_engine** out) {
    if (!d || !out || n_devices < 1 || !d->site_xyz || !d->site_kind || !d->tri_xyz || !d->face_sphere ||
        !d->list_offsets || (!d->list_faces && d->list_offsets[d->n_sites] > 0)) {
        set_err("p2m_engine_create: invalid descriptor");
        return P2M_ERR_INVALID;
    }
    if (d->n_sites == 0 || d->n_faces == 0 || d->n_sites >= (1ull << 32) || d->n_faces >= (1ull << 32)) {
        set_err("p2m_engine_create: engine not built (no sites/faces) or too large");
        return P2M_ERR_NOT_BUILT;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        set_err("p2m_engine_create: no CUDA device available");
        return P2M_ERR_CUDA;
    }
    const uint64_t S = d->n_sites, F = d->n_faces, L = d->list_offsets[S];
    for (uint64_t s = 0; s < S; ++s)
        if (d->list_offsets[s] > d->list_offsets[s + 1]) { set_err("p2m_engine_create: offsets not monotone"); return P2M_ERR_INVALID; }
    for (uint64_t j = 0; j < L; ++j)
        if (d->list_faces[j] >= F) { set_err("p2m_engine_create: list face id out of range"); return P2M_ERR_INVALID; }

    auto E = std::make_unique<p2m_engine>();
    E->n_sites = S; E->n_faces = F; E->n_entries = L;
    if (d->adj_offsets && d->adj_sites) {
        if (d->adj_offsets[0] != 0) { set_err("p2m_engine_create: adjacency offsets must start at 0"); return P2M_ERR_INVALID; }
        for (uint64_t s = 0; s < S; ++s)
            if (d->adj_offsets[s] > d->adj_offsets[s + 1]) { set_err("p2m_engine_create: adjacency offsets not monotone"); return P2M_ERR_INVALID; }
        for (uint64_t k = 0; k < d->adj_offsets[S]; ++k)
            if (d->adj_sites[k] >= S) { set_err("p2m_engine_create: adjacency site id out of range"); return P2M_ERR_INVALID; }
        E->has_adj = true;
        E->n_adj = d->adj_offsets[S];
    }

    // ---- pack ----
    std::vector<uint32_t> node_site;
    std::vector<uint8_t> node_dim;
    build_kdtree(d->site_xyz, S, node_site, node_dim);
    std::vector<D4> kd(S);
    double klo[3] = {INFINITY, INFINITY, INFINITY}, khi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint64_t k = 0; k < S; ++k) {
        const uint32_t id = node_site[k];
        const double* p = d->site_xyz + 3 * (uint64_t)id;
        uint64_t meta = (uint64_t)id | (uint64_t)node_dim[k] << 32 |
                        (d->site_kind[id] == P2M_SITE_SENTINEL ? (1ull << 34) : 0ull);
        kd[k] = D4{p[0], p[1], p[2], bits_to_double(meta)};
        if (d->site_kind[id] != P2M_SITE_SENTINEL)
            for (int c = 0; c < 3; ++c) { klo[c] = std::min(klo[c], p[c]); khi[c] = std::max(khi[c], p[c]); }
    }
    std::vector<D4> rec(4 * F);
    for (uint64_t f = 0; f < F; ++f) {
        const double* t = d->tri_xyz + 9 * f;
        const double* s = d->face_sphere + 4 * f;
        rec[4 * f] = D4{s[0], s[1], s[2], s[3]};
        rec[4 * f + 1] = D4{t[0], t[1], t[2], t[3]};
        rec[4 * f + 2] = D4{t[4], t[5], t[6], t[7]};
        // padding of the last sector: the face's unit normal in fp32 (for the plane-distance bound)
        const double ux = t[3] - t[0], uy = t[4] - t[1], uz = t[5] - t[2];
        const double vx = t[6] - t[0], vy = t[7] - t[1], vz = t[8] - t[2];
        double nx = uy * vz - uz * vy, ny = uz * vx - ux * vz, nz = ux * vy - uy * vx;
        const double nl = std::sqrt(nx * nx + ny * ny + nz * nz);
        if (nl > 0.0 && std::isfinite(nl)) { nx /= nl; ny /= nl; nz /= nl; } else { nx = ny = nz = 0.0; }
        const float fn[4] = {(float)nx, (float)ny, (float)nz, 0.0f};
        double p0, p1;
        std::memcpy(&p0, fn, 8);
        std::memcpy(&p1, fn + 2, 8);
        rec[4 * f + 3] = D4{t[8], p0, p1, 0.0};
    }
    // fp32 bound of the scan's level 2: each face's bounding disk (a cylinder of height ~0 around its
    // min-enclosing-sphere centre), DESIGN.md section 9.  M = max |coordinate| of D scales the
    // device's fp32 error terms.
    double Mdom = 0.0;
    for (int c = 0; c < 3; ++c) Mdom = std::max({Mdom, std::fabs(d->domain_min[c]), std::fabs(d->domain_max[c])});
    std::vector<float4> fcy(kCy * F);
    auto group_normal = [&](const uint32_t* ids, uint64_t k, double* nsum, std::vector<double>& pts) {
        nsum[0] = nsum[1] = nsum[2] = 0.0;
        pts.resize(9 * k);
        for (uint64_t i = 0; i < k; ++i) {
            const double* t = d->tri_xyz + 9 * (uint64_t)(ids ? ids[i] : i);
            for (int c = 0; c < 9; ++c) pts[9 * i + c] = t[c];
            const double ux = t[3] - t[0], uy = t[4] - t[1], uz = t[5] - t[2];
            const double vx = t[6] - t[0], vy = t[7] - t[1], vz = t[8] - t[2];
            nsum[0] += uy * vz - uz * vy; nsum[1] += uz * vx - ux * vz; nsum[2] += ux * vy - uy * vx;
        }
    };
    parallel_sites(F, [&](uint64_t f0, uint64_t f1) {
        std::vector<double> pts;
        double ns[3];
        for (uint64_t f = f0; f < f1; ++f) {
            const uint32_t id = (uint32_t)f;
            group_normal(&id, 1, ns, pts);
            fit_cyl(pts.data(), 3, ns, d->face_sphere + 4 * f, fcy.data() + kCy * f);
        }
    });
    // The disk centre is the face's min-enclosing-circle centre (the circumcentre of an acute face, the
    // midpoint of the longest edge otherwise): a point of the face up to rounding.  The largest distance
    // from a stored fp32 centre to its face makes |q - c| an upper bound of d(q, face) (scan d_min).
    double ctr_slack = 0.0;
    {
        std::vector<double> part(F ? F : 1, 0.0);
        parallel_sites(F, [&](uint64_t f0, uint64_t f1) {
            for (uint64_t f = f0; f < f1; ++f) {
                const double* t = d->tri_xyz + 9 * f;
                const float4 c = fcy[kCy * f];
                p2m::V3 cp;
                part[f] = std::sqrt(p2m::closest_tri(p2m::V3{c.x, c.y, c.z}, p2m::ld3(t), p2m::ld3(t + 3), p2m::ld3(t + 6), &cp));
            }
        });
        for (double v : part) ctr_slack = std::max(ctr_slack, v);
        ctr_slack = ctr_slack * (1.0 + 1e-9) + 1e-12 * Mdom;
    }
    // Spatial list order for the grouped scan (lfs): the (d^2, face id) argmin does not depend on
    // the order a list is scanned in, so each list is re-sorted by the Morton code of its faces'
    // sphere centres (ties by id) -- its 32-entry batches and 256-entry chunks then enclose compact
    // surface patches and their spheres prune whole.  lf keeps the ascending order of
    // REF/SPEC.md:392 for the sequential fused path (oracle-identical counters).
    std::vector<uint32_t> lfs(std::max<uint64_t>(1, L));
    {
        double clo[3] = {INFINITY, INFINITY, INFINITY}, chi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (uint64_t f = 0; f < F; ++f)
            for (int k = 0; k < 3; ++k) {
                clo[k] = std::min(clo[k], d->face_sphere[4 * f + k]);
                chi[k] = std::max(chi[k], d->face_sphere[4 * f + k]);
            }
        std::vector<uint64_t> fkey(F);
        auto spread = [](uint64_t x) {  // 21 bits -> every third bit
            x &= 0x1fffff;
            x = (x | x << 32) & 0x1f00000000ffffull;
            x = (x | x << 16) & 0x1f0000ff0000ffull;
            x = (x | x << 8) & 0x100f00f00f00f00full;
            x = (x | x << 4) & 0x10c30c30c30c30c3ull;
            x = (x | x << 2) & 0x1249249249249249ull;
            return x;
        };
        for (uint64_t f = 0; f < F; ++f) {
            uint64_t key = 0;
            for (int k = 0; k < 3; ++k) {
                const double ext = chi[k] - clo[k];
                const double t = ext > 0 ? (d->face_sphere[4 * f + k] - clo[k]) / ext : 0.0;
                key |= spread((uint64_t)std::min(2097151.0, std::max(0.0, t * 2097152.0))) << k;
            }
            fkey[f] = key;
        }
        const bool spatial = std::getenv("P2M_NO_SPATIAL") == nullptr;
        parallel_sites(S, [&](uint64_t s0, uint64_t s1) {
            std::vector<std::pair<uint64_t, uint32_t>> tmp;
            for (uint64_t s = s0; s < s1; ++s) {
                const uint64_t b0 = d->list_offsets[s], b1 = d->list_offsets[s + 1];
                tmp.clear();
                for (uint64_t j = b0; j < b1; ++j) tmp.push_back({spatial ? fkey[d->list_faces[j]] : 0ull, d->list_faces[j]});
                std::sort(tmp.begin(), tmp.end());
                for (uint64_t j = b0; j < b1; ++j) lfs[j] = tmp[j - b0].second;
            }
        });
    }
    // d_min seed points over lfs, one per aligned 32-entry batch and one per aligned 256-entry chunk:
    // a point ON the mesh near the group's centre (the closest point of the member faces to the centre
    // of their sphere boxes), rounded to fp32 -- |q - P| + the rounding slack bounds d(q, M) from above
    auto group_point = [&](uint64_t j, uint64_t je) {
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (uint64_t t = j; t < je; ++t) {
            const double* sp = d->face_sphere + 4 * (uint64_t)lfs[t];
            for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], sp[k] - sp[3]); hi[k] = std::max(hi[k], sp[k] + sp[3]); }
        }
        const p2m::V3 C{0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
        double bd = INFINITY;
        p2m::V3 P{0, 0, 0};
        for (uint64_t t = j; t < je; ++t) {
            const double* tr = d->tri_xyz + 9 * (uint64_t)lfs[t];
            p2m::V3 cp;
            const double dd = p2m::closest_tri(C, p2m::ld3(tr), p2m::ld3(tr + 3), p2m::ld3(tr + 6), &cp);
            if (dd < bd) { bd = dd; P = cp; }
        }
        return make_float4((float)P.x, (float)P.y, (float)P.z, 0.0f);
    };
    std::vector<uint64_t> boff(S + 1, 0), coff(S + 1, 0);
    for (uint64_t s = 0; s < S; ++s) {
        const uint64_t len = d->list_offsets[s + 1] - d->list_offsets[s];
        boff[s + 1] = boff[s] + (len + 31) / 32;
        coff[s + 1] = coff[s] + (len + kListChunk - 1) / kListChunk;
    }
    E->n_batches = boff[S];
    E->n_chunks = coff[S];
    std::vector<float4> bpt(std::max<uint64_t>(1, E->n_batches)), cpt(std::max<uint64_t>(1, E->n_chunks));
    std::vector<float4> bcy(kCy * std::max<uint64_t>(1, E->n_batches)), ccy(kCy * std::max<uint64_t>(1, E->n_chunks));
    parallel_sites(S, [&](uint64_t s0, uint64_t s1) {
        std::vector<double> pts;
        double ns[3];
        for (uint64_t s = s0; s < s1; ++s) {
            const uint64_t b0 = d->list_offsets[s], b1 = d->list_offsets[s + 1];
            for (uint64_t j = b0, bi = boff[s]; j < b1; j += 32, ++bi) {
                const uint64_t je = std::min(b1, j + 32);
                bpt[bi] = group_point(j, je);
                group_normal(lfs.data() + j, je - j, ns, pts);
                fit_cyl(pts.data(), (int)(3 * (je - j)), ns, nullptr, bcy.data() + kCy * bi);
            }
            for (uint64_t j = b0, ci = coff[s]; j < b1; j += kListChunk, ++ci) {
                const uint64_t je = std::min(b1, j + kListChunk);
                cpt[ci] = group_point(j, je);
                group_normal(lfs.data() + j, je - j, ns, pts);
                fit_cyl(pts.data(), (int)(3 * (je - j)), ns, nullptr, ccy.data() + kCy * ci);
            }
        }
    });
    FlatBvh bvh;
    build_bvh(d->tri_xyz, F, bvh);
    E->n_bvh = bvh.nodes.size() / 2;

    Params P{};
    P.n_nodes = (uint32_t)S;
    P.n_faces = (uint32_t)F;
    double dd2 = 0.0;
    {
        double dx = d->domain_max[0] - d->domain_min[0], dy = d->domain_max[1] - d->domain_min[1],
               dz = d->domain_max[2] - d->domain_min[2];
        dd2 = dx * dx + dy * dy + dz * dz;
    }
    P.prune_eps = 1e-9 * std::sqrt(dd2);  // same definition as the oracle (orc_ctx_create)
    {
        // fp32 error scale of the scan's bounds: the largest |coordinate| of the mesh and of every
        // stored centre / point; the kernels take max(|q|, mesh_m) per row
        float mm = 0.f;
        for (uint64_t i = 0; i < 3 * F; ++i) mm = std::max(mm, round_up_f(std::fabs(d->tri_xyz[i])));
        auto scan4 = [&](const std::vector<float4>& v, int stride) {
            for (size_t i = 0; i < v.size(); i += stride) mm = std::max({mm, std::fabs(v[i].x), std::fabs(v[i].y), std::fabs(v[i].z)});
        };
        scan4(fcy, kCy); scan4(bcy, kCy); scan4(ccy, kCy); scan4(bpt, 1); scan4(cpt, 1);
        P.mesh_m = mm;
        P.eps2 = round_up_f(2.0 * P.prune_eps);
        P.ctr_slack = round_up_f(ctr_slack);
    }
    P.long_tile = 32;
    if (const char* v = std::getenv("P2M_LONG_TILE")) {
        uint32_t t = (uint32_t)std::strtoul(v, nullptr, 10);
        if (t == 32 || t == 64 || t == 128 || t == 256) P.long_tile = t;
    }
    double kext[3] = {0, 0, 0};  // Morton key box = cell-locate grid box extents
    for (int c = 0; c < 3; ++c) {
        P.dmin[c] = d->domain_min[c];
        P.dmax[c] = d->domain_max[c];
        if (!(klo[c] <= khi[c])) { klo[c] = d->domain_min[c]; khi[c] = d->domain_max[c]; }
        double mid = 0.5 * (klo[c] + khi[c]), h = 0.75 * (khi[c] - klo[c]);  // = builder.cpp gbox
        if (!(h > 0)) h = 1.0;
        P.key_lo[c] = mid - h;
        P.key_scale[c] = 1024.0 / (2.0 * h);
        kext[c] = 2.0 * h;
    }

    Grid grid;
    {
        double ext[3];
        for (int c = 0; c < 3; ++c) ext[c] = kext[c];
        if (build_grid(d, P.key_lo, ext, grid, kd, device_ids ? device_ids[0] : 0)) {
            E->grid_cells = (uint64_t)grid.res[0] * grid.res[1] * grid.res[2];
            E->grid_pairs = grid.site.size();
            for (int c = 0; c < 3; ++c) { P.grid_lo[c] = grid.lo[c]; P.grid_inv[c] = grid.inv[c]; P.grid_res[c] = grid.res[c]; }
        }
        if (std::getenv("P2M_NO_GRID")) E->grid_cells = E->grid_pairs = 0;
        P.no_seed = std::getenv("P2M_NO_SEED") ? 1 : std::getenv("P2M_NO_DEEP_SEED") ? 2 : 0;  // 2: group-point seeds only
        P.no_batch = std::getenv("P2M_NO_BATCH") ? 1 : 0;
    }
    std::vector<D4> site_pos(S), site_ref(S);
    for (uint64_t i = 0; i < S; ++i) {
        const double* x = d->site_xyz + 3 * i;
        site_pos[i] = D4{x[0], x[1], x[2], bits_to_double(d->site_kind[i] == P2M_SITE_SENTINEL ? (1ull << 34) : 0ull)};
        // a point on the mesh for the d_min seed: the vertex itself, or the auxiliary projection
        site_ref[i] = D4{0.0, 0.0, 0.0, 0.0};
        if (d->site_kind[i] == P2M_SITE_MESH_VERTEX) {
            site_ref[i] = D4{x[0], x[1], x[2], 1.0};
        } else if (d->site_kind[i] == P2M_SITE_AUXILIARY && d->site_ref_xyz) {
            const double* r = d->site_ref_xyz + 3 * i;
            if (std::isfinite(r[0]) && std::isfinite(r[1]) && std::isfinite(r[2])) site_ref[i] = D4{r[0], r[1], r[2], 1.0};
        }
    }
    // ---- upload to the first device, peer-replicate to the rest ----
    Image I;
    I.kd.set(kd.data(), S); I.rec.set(rec.data(), 4 * F); I.fcy.set(fcy.data(), fcy.size());
    I.bpt.set(bpt.data(), bpt.size()); I.boff.set(boff.data(), S + 1);
    I.bcy.set(bcy.data(), bcy.size()); I.ccy.set(ccy.data(), ccy.size());
    I.off.set(d->list_offsets, S + 1); I.lf.set(d->list_faces, L); I.lfs.set(lfs.data(), L);
    I.cpt.set(cpt.data(), cpt.size()); I.coff.set(coff.data(), S + 1);
    I.bvh.set(bvh.nodes.data(), bvh.nodes.size()); I.bvh_perm.set(bvh.perm.data(), F);
    I.site_pos.set(site_pos.data(), S); I.site_ref.set(site_ref.data(), S);
    if (E->has_adj) { I.adj_off.set(d->adj_offsets, S + 1); I.adj.set(d->adj_sites, E->n_adj); }
    if (E->grid_cells) { I.grid_off.set(grid.off.data(), E->grid_cells + 1); I.grid_site.set(grid.site.data(), E->grid_pairs); }
    auto fail = [&](int rc) { for (auto& x : E->slots) free_slot(*x); return rc; };
    {
        int rc = upload_engine(E.get(), P, I, n_devices, device_ids, ndev);
        if (rc != P2M_OK) return fail(rc);
        rc = mark_heavy_sites(E.get(), d->site_xyz, d->site_kind);
        if (rc != P2M_OK) return fail(rc);
        E->bytes += S;                           // the heavy-site flags (not part of the packed image)
    }
    *out = E.release();
    return P2M_OK;
}

// ---- device image file "P2MD" (p2m_engine_save / p2m_engine_load) ---------------------------------
// Little-endian.  magic "P2MD", u32 version, then the engine counts (u64 each), the kernel parameters
// field by field (fixed widths), then every array of the Image as (u64 byte count, bytes) in a fixed
// order, then an FNV-1a 64 checksum of everything before it.  Load validates counts, sizes, CSR
// monotonicity and every stored id against its range before anything reaches a device.
namespace {

constexpr uint32_t kImageVersion = 2;  // v2: bounding cylinders (fcy/bcy/ccy) replace the v1 sphere/plane records

struct Fnv {
    uint64_t h = 1469598103934665603ull;
    void add(const void* p, size_t n) {
        const unsigned char* c = (const unsigned char*)p;
        for (size_t i = 0; i < n; ++i) { h ^= c[i]; h *= 1099511628211ull; }
    }
};

struct Writer {
    FILE* fp;
    Fnv fnv;
    bool ok = true;
    void put(const void* p, size_t n) {
        if (!ok || !n) return;
        fnv.add(p, n);
        ok = std::fwrite(p, 1, n, fp) == n;
    }
    template <class T> void v(T x) { put(&x, sizeof x); }
};

struct Reader {
    FILE* fp;
    Fnv fnv;
    bool ok = true;
    void get(void* p, size_t n) {
        if (!ok || !n) return;
        ok = std::fread(p, 1, n, fp) == n;
        if (ok) fnv.add(p, n);
    }
    template <class T> T v() { T x{}; get(&x, sizeof x); return x; }
};

// the scalar fields of Params that describe the layout (pointers are re-derived on upload)
template <class IO, class F>
void params_fields(Params& P, F&& f) {
    for (int c = 0; c < 3; ++c) { f(P.dmin[c]); f(P.dmax[c]); f(P.key_lo[c]); f(P.key_scale[c]); f(P.grid_lo[c]); f(P.grid_inv[c]); f(P.grid_res[c]); }
    f(P.prune_eps); f(P.mesh_m); f(P.eps2); f(P.ctr_slack); f(P.long_tile); f(P.no_seed); f(P.no_batch); f(P.n_nodes); f(P.n_faces);
}

template <class T>
bool all_below(const T* p, uint64_t n, uint64_t lim) {
    for (uint64_t i = 0; i < n; ++i) if ((uint64_t)p[i] >= lim) return false;
    return true;
}
template <class T>
bool csr_ok(const T* off, uint64_t n, uint64_t total) {
    if (off[0] != 0 || (uint64_t)off[n] != total) return false;
    for (uint64_t i = 0; i < n; ++i) if (off[i] > off[i + 1]) return false;
    return true;
}

}  // namespace

P2M_API int p2m_engine_save(const p2m_engine* e, const char* path) {
    if (!e || e->slots.empty()) { set_err("p2m_engine_save: engine not built"); return P2M_ERR_NOT_BUILT; }
    if (!path) { set_err("p2m_engine_save: null path"); return P2M_ERR_INVALID; }
    const Slot& s = *e->slots[0];
    const uint64_t S = e->n_sites, F = e->n_faces, L = e->n_entries;
    CK(cudaSetDevice(s.dev));
    CK(cudaDeviceSynchronize());
    struct A { const void* dev; uint64_t bytes; };
    const A arrs[] = {
        {s.kd, 32 * S}, {s.rec, 128 * F}, {s.fcy, 16ull * kCy * F}, {s.bcy, 16ull * kCy * e->n_batches},
        {s.ccy, 16ull * kCy * e->n_chunks}, {s.bpt, 16 * e->n_batches}, {s.boff, 8 * (S + 1)}, {s.off, 8 * (S + 1)}, {s.lf, 4 * L}, {s.lfs, 4 * L}, {s.cpt, 16 * e->n_chunks},
        {s.coff, 8 * (S + 1)}, {s.bvh, 64 * e->n_bvh}, {s.bvh_perm, 4 * F}, {s.site_pos, 32 * S}, {s.site_ref, 32 * S},
        {s.adj_off, e->has_adj ? 8 * (S + 1) : 0}, {s.adj, e->has_adj ? 4 * e->n_adj : 0},
        {s.grid_off, e->grid_cells ? 4 * (e->grid_cells + 1) : 0}, {s.grid_site, e->grid_cells ? 4 * e->grid_pairs : 0},
        {s.heavy, S}};
    FILE* fp = std::fopen(path, "wb");
    if (!fp) { set_err(std::string("p2m_engine_save: cannot open ") + path); return P2M_ERR_IO; }
    Writer w{fp};
    w.put("P2MD", 4);
    w.v<uint32_t>(kImageVersion);
    const uint64_t counts[12] = {S, F, L, e->n_batches, e->n_chunks, e->n_bvh, e->grid_cells, e->grid_pairs,
                                 (uint64_t)e->has_adj, e->n_adj, e->n_heavy, 0};
    for (uint64_t c : counts) w.v<uint64_t>(c);
    Params P = s.params;
    params_fields<Writer>(P, [&](auto& x) { w.v(x); });
    std::vector<unsigned char> buf;
    for (const A& a : arrs) {
        w.v<uint64_t>(a.bytes);
        if (!a.bytes) continue;
        buf.resize(a.bytes);
        if (cudaMemcpy(buf.data(), a.dev, a.bytes, cudaMemcpyDeviceToHost) != cudaSuccess) {
            std::fclose(fp);
            set_err("p2m_engine_save: device read failed");
            return P2M_ERR_CUDA;
        }
        w.put(buf.data(), a.bytes);
    }
    const uint64_t sum = w.fnv.h;
    w.ok = w.ok && std::fwrite(&sum, 8, 1, fp) == 1;
    const bool ok = w.ok && std::fclose(fp) == 0;
    if (!ok) { set_err("p2m_engine_save: write failed"); return P2M_ERR_IO; }
    return P2M_OK;
}

P2M_API int p2m_engine_load(const char* path, int n_devices, const int* device_ids, p2m_engine** out) {
    if (!path || !out || n_devices < 1) { set_err("p2m_engine_load: invalid argument"); return P2M_ERR_INVALID; }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        set_err("p2m_engine_load: no CUDA device available");
        return P2M_ERR_CUDA;
    }
    FILE* fp = std::fopen(path, "rb");
    if (!fp) { set_err(std::string("p2m_engine_load: cannot open ") + path); return P2M_ERR_IO; }
    Reader r{fp};
    auto bad = [&](const char* why) { std::fclose(fp); set_err(std::string("p2m_engine_load: ") + why); return (int)P2M_ERR_IO; };
    char magic[4] = {0, 0, 0, 0};
    r.get(magic, 4);
    if (!r.ok || std::memcmp(magic, "P2MD", 4) != 0) return bad("not a device image (magic)");
    if (r.v<uint32_t>() != kImageVersion || !r.ok) return bad("device image version mismatch");
    uint64_t c[12];
    for (auto& x : c) x = r.v<uint64_t>();
    if (!r.ok) return bad("truncated (header)");
    auto E = std::make_unique<p2m_engine>();
    E->n_sites = c[0]; E->n_faces = c[1]; E->n_entries = c[2]; E->n_batches = c[3]; E->n_chunks = c[4];
    E->n_bvh = c[5]; E->grid_cells = c[6]; E->grid_pairs = c[7]; E->has_adj = c[8] != 0; E->n_adj = c[9];
    E->n_heavy = c[10];
    const uint64_t S = c[0], F = c[1], L = c[2];
    if (S == 0 || F == 0 || S >= (1ull << 32) || F >= (1ull << 32) || L >= (1ull << 40) || c[3] > L + S ||
        c[4] > L + S || c[5] == 0 || c[5] > 4 * F || c[6] > (1ull << 30) || c[7] >= (1ull << 36) || c[8] > 1 ||
        c[9] >= (1ull << 36) || c[10] > S)
        return bad("implausible counts");
    Params P{};
    params_fields<Reader>(P, [&](auto& x) { x = r.v<std::remove_reference_t<decltype(x)>>(); });
    if (!r.ok) return bad("truncated (parameters)");
    if (P.n_nodes != S || P.n_faces != F) return bad("parameters do not match the counts");
    Image I;
    bool sizes_ok = true;
    auto rd = [&](auto& arr, uint64_t n) {
        using T = typename std::remove_reference_t<decltype(arr.own)>::value_type;
        const uint64_t bytes = r.v<uint64_t>();
        if (!r.ok || bytes != sizeof(T) * n) { sizes_ok = false; return; }
        std::vector<T> v(n);
        r.get(v.data(), bytes);
        arr.take(std::move(v));
    };
    rd(I.kd, S); rd(I.rec, 4 * F); rd(I.fcy, (uint64_t)kCy * F); rd(I.bcy, (uint64_t)kCy * E->n_batches);
    rd(I.ccy, (uint64_t)kCy * E->n_chunks); rd(I.bpt, E->n_batches); rd(I.boff, S + 1); rd(I.off, S + 1); rd(I.lf, L); rd(I.lfs, L); rd(I.cpt, E->n_chunks);
    rd(I.coff, S + 1); rd(I.bvh, 2 * E->n_bvh); rd(I.bvh_perm, F); rd(I.site_pos, S); rd(I.site_ref, S);
    rd(I.adj_off, E->has_adj ? S + 1 : 0); rd(I.adj, E->has_adj ? E->n_adj : 0);
    rd(I.grid_off, E->grid_cells ? E->grid_cells + 1 : 0); rd(I.grid_site, E->grid_cells ? E->grid_pairs : 0);
    rd(I.heavy, S);
    if (!sizes_ok || !r.ok) return bad("truncated or inconsistent array sizes");
    uint64_t sum = 0;
    if (std::fread(&sum, 8, 1, fp) != 1 || sum != r.fnv.h) return bad("checksum mismatch (corrupt file)");
    std::fclose(fp);
    // ranges of every stored id / offset (a corrupt or foreign file must not reach the kernels)
    auto inval = [&](const char* why) { set_err(std::string("p2m_engine_load: invalid image: ") + why); return (int)P2M_ERR_IO; };
    if (!csr_ok(I.off.p, S, L)) return inval("list offsets");
    if (!all_below(I.lf.p, L, F) || !all_below(I.lfs.p, L, F)) return inval("list face ids");
    if (!csr_ok(I.boff.p, S, E->n_batches) || !csr_ok(I.coff.p, S, E->n_chunks)) return inval("group offsets");
    for (uint64_t i = 0; i < S; ++i) {
        const uint64_t len = I.off.p[i + 1] - I.off.p[i];
        if (I.boff.p[i + 1] - I.boff.p[i] != (len + 31) / 32 || I.coff.p[i + 1] - I.coff.p[i] != (len + kListChunk - 1) / kListChunk)
            return inval("group offsets do not match the lists");
    }
    for (uint64_t k = 0; k < S; ++k) {
        uint64_t meta;
        std::memcpy(&meta, &I.kd.p[k].w, 8);
        if ((meta & 0xffffffffull) >= S || ((meta >> 32) & 3) > 2) return inval("k-d nodes");
    }
    if (!all_below(I.bvh_perm.p, F, F)) return inval("bvh leaf ids");
    for (uint64_t k = 0; k < E->n_bvh; ++k) {
        uint64_t meta;
        std::memcpy(&meta, &I.bvh.p[2 * k + 1].z, 8);
        const uint64_t cnt = meta >> 32, first = meta & 0xffffffffull;
        if (cnt ? (first + cnt > F || cnt > 4) : (first == 0 || first >= E->n_bvh)) return inval("bvh nodes");
    }
    if (E->has_adj && (!csr_ok(I.adj_off.p, S, E->n_adj) || !all_below(I.adj.p, E->n_adj, S))) return inval("adjacency");
    if (E->grid_cells) {
        if (!csr_ok(I.grid_off.p, E->grid_cells, E->grid_pairs) || !all_below(I.grid_site.p, E->grid_pairs, S))
            return inval("cell-locate grid");
        if ((uint64_t)P.grid_res[0] * P.grid_res[1] * P.grid_res[2] != E->grid_cells) return inval("grid resolution");
    }
    if (!all_below(I.heavy.p, S, 2)) return inval("heavy flags");
    auto fail = [&](int rc) { for (auto& x : E->slots) free_slot(*x); return rc; };
    int rc = upload_engine(E.get(), P, I, n_devices, device_ids, ndev);
    if (rc != P2M_OK) return fail(rc);
    *out = E.release();
    return P2M_OK;
}

P2M_API void p2m_engine_destroy(p2m_engine* e) {
    if (!e) return;
    for (auto& s : e->slots) free_slot(*s);
    delete e;
}

P2M_API int p2m_engine_info(const p2m_engine* e, int* n, double* ms, uint64_t* bytes) {
    if (!e) { set_err("p2m_engine_info: engine not built"); return P2M_ERR_NOT_BUILT; }
    if (n) *n = (int)e->slots.size();
    if (ms) *ms = e->replicate_ms;
    if (bytes) *bytes = e->bytes;
    return P2M_OK;
}

P2M_API int p2m_query_device(p2m_engine* e, int slot, const double* d_q, uint64_t n, double* d_dist, double* d_cp,
                             uint32_t* d_face, uint32_t* d_site, uint32_t* d_flags, void* stream, p2m_counters* cnt) {
    if (!e) { set_err("p2m_query_device: engine not built"); return P2M_ERR_NOT_BUILT; }
    if (slot < 0 || slot >= (int)e->slots.size()) { set_err("p2m_query_device: bad slot"); return P2M_ERR_INVALID; }
    if (n && (!d_q || !d_dist || !d_cp || !d_face || !d_site)) { set_err("p2m_query_device: null buffer"); return P2M_ERR_INVALID; }
    Slot& s = *e->slots[slot];
    cudaStream_t st = (cudaStream_t)stream;
    if (cnt) std::memset(cnt, 0, sizeof *cnt);
    if (!n) return P2M_OK;
    p2m::dev::Out o{d_dist, d_cp, d_face, d_site, d_flags, nullptr, nullptr};
    std::unique_lock<std::mutex> lk(s.mu, std::defer_lock);
    if (cnt) {
        lk.lock();
        CK(cudaSetDevice(s.dev));
        CK(cudaMemsetAsync(s.agg, 0, sizeof(unsigned long long) * 8, st));
        o.agg = s.agg;
    }
    int rc = run_pipeline(e, s, d_q, n, o, cnt != nullptr, st, false, nullptr);
    if (rc != P2M_OK) return rc;
    if (cnt) {
        unsigned long long h[8];
        CK(cudaMemcpyAsync(h, s.agg, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cnt->n_queries = n;
        cnt->candidates_visited = h[0];
        cnt->exact_evaluations = h[1];
        cnt->pruned = h[0] - h[1];
        cnt->kd_nodes_visited = h[2];
        cnt->filter_passes = h[4];
        cnt->warp_rare_iters = h[5];
        cnt->structure_bytes = h[6];
        cnt->scan_tiles = h[7];
        cnt->fallbacks = h[3];
    }
    return P2M_OK;
}

P2M_API int p2m_nearest_site_device(p2m_engine* e, int slot, const double* d_q, uint64_t n, uint32_t* d_site, void* stream) {
    if (!e) { set_err("p2m_nearest_site_device: engine not built"); return P2M_ERR_NOT_BUILT; }
    if (slot < 0 || slot >= (int)e->slots.size()) { set_err("bad slot"); return P2M_ERR_INVALID; }
    if (!n) return P2M_OK;
    p2m::dev::Out o{};
    return run_pipeline(e, *e->slots[slot], d_q, n, o, false, (cudaStream_t)stream, true, d_site);
}

P2M_API int p2m_query_device_counters(p2m_engine* e, int slot, const double* d_q, uint64_t n, uint64_t* d_pq, void* stream) {
    if (!e) { set_err("p2m_query_device_counters: engine not built"); return P2M_ERR_NOT_BUILT; }
    if (slot < 0 || slot >= (int)e->slots.size()) { set_err("bad slot"); return P2M_ERR_INVALID; }
    if (!n) return P2M_OK;
    Slot& s = *e->slots[slot];
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaSetDevice(s.dev));
    double *dist = nullptr, *cp = nullptr;
    uint32_t *face = nullptr, *site = nullptr;
    CK(cudaMallocAsync(&dist, 8 * n, st));
    CK(cudaMallocAsync(&cp, 24 * n, st));
    CK(cudaMallocAsync(&face, 4 * n, st));
    CK(cudaMallocAsync(&site, 4 * n, st));
    p2m::dev::Out o{dist, cp, face, site, nullptr, d_pq, nullptr};
    int rc = run_pipeline(e, s, d_q, n, o, true, st, false, nullptr);
    cudaFreeAsync(dist, st); cudaFreeAsync(cp, st); cudaFreeAsync(face, st); cudaFreeAsync(site, st);
    return rc;
}

// true if the host pointer is page-locked (cudaHostAlloc / cudaHostRegister) -- the DMA engines can
// read or write it asynchronously; pageable memory goes through the bounce rings
bool host_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int ensure_bounce(Slot& s) {
    auto& b = s.bnc;
    if (b.ready) return P2M_OK;
    for (int k = 0; k < Slot::Bounce::kIn; ++k) {
        CK(cudaHostAlloc((void**)&b.in[k], 24 * Slot::Bounce::kRows, cudaHostAllocPortable));
        CK(cudaEventCreateWithFlags(&b.in_ev[k], cudaEventDisableTiming));
    }
    for (int k = 0; k < Slot::Bounce::kOut; ++k) {
        CK(cudaHostAlloc((void**)&b.out[k], 44 * Slot::Bounce::kRows, cudaHostAllocPortable));
        CK(cudaEventCreateWithFlags(&b.out_ev[k], cudaEventDisableTiming));
    }
    const int hw = (int)std::max(2u, std::thread::hardware_concurrency());
    b.pack.reset(new CopyPool(std::min(3, hw / 4)));
    b.unpack.reset(new CopyPool(std::min(5, hw / 3)));
    b.ready = true;
    return P2M_OK;
}

// The host-buffer pipeline for pageable caller arrays (p2m_query): the same chunk schedule, device
// staging sets and streams as the pinned path; every H2D/D2H copy goes through a pinned bounce
// sub-chunk.  This thread: pack input sub-chunks + enqueue H2D, then the chunk's kernels.  Output
// thread: per finished chunk, enqueue D2H sub-copies into the out-ring, unpack completed ones.
int run_bounce(p2m_engine* e, Slot& s, const double* q, double* dist, double* cp, uint32_t* face, uint32_t* site,
               uint32_t* flags, uint64_t b, const std::vector<uint64_t>& len_of, p2m_counters* cnt,
               p2m_counters& part, bool serial_kernels) {
    using B = Slot::Bounce;
    auto& bn = s.bnc;
    const size_t nch = len_of.size();
    std::vector<uint64_t> start(nch);
    for (size_t c = 0, o = 0; c < nch; ++c) { start[c] = o; o += len_of[c]; }
    std::mutex mu;
    std::condition_variable cv;
    size_t launched = 0, drained = 0;  // chunks whose kernels are enqueued / whose D2H copies are enqueued
    int out_rc = P2M_OK;
    std::string out_err;
    std::thread out([&] {
        int rc = P2M_OK;
        auto fail = [&](int r) { rc = r; out_err = p2m_last_error(); };
        if (cudaSetDevice(s.dev) != cudaSuccess) { set_err("cudaSetDevice"); fail(P2M_ERR_CUDA); }
        struct Pend { uint64_t r0 = 0, len = 0; bool live = false; } pend[B::kOut];
        auto unpack = [&](int k) {
            Pend& p = pend[k];
            if (!p.live) return (int)P2M_OK;
            if (cudaEventSynchronize(bn.out_ev[k]) != cudaSuccess) { set_err("bounce D2H failed"); return (int)P2M_ERR_CUDA; }
            const unsigned char* o = bn.out[k];
            const uint64_t L = p.len, r = b + p.r0;
            const CopyPool::Seg segs[5] = {{dist + r, o, 8 * L}, {cp + 3 * r, o + 8 * B::kRows, 24 * L},
                                           {face + r, o + 32 * B::kRows, 4 * L}, {site + r, o + 36 * B::kRows, 4 * L},
                                           {flags ? flags + r : nullptr, o + 40 * B::kRows, flags ? 4 * L : 0}};
            bn.unpack->run(segs, 5);
            p.live = false;
            return (int)P2M_OK;
        };
        uint64_t j = 0;
        for (size_t c = 0; c < nch && rc == P2M_OK; ++c) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return launched > c || out_rc != P2M_OK; });
                if (out_rc != P2M_OK) break;
            }
            const Slot::Ws& w = s.ws[c % Slot::kPipe];
            if (cudaStreamWaitEvent(s.d2h, s.cev[3 * c + 1], 0) != cudaSuccess) { set_err("d2h wait"); fail(P2M_ERR_CUDA); break; }
            for (uint64_t o = 0; o < len_of[c] && rc == P2M_OK; o += B::kRows, ++j) {
                const int k = (int)(j % B::kOut);
                int r2 = unpack(k);
                if (r2 != P2M_OK) { fail(r2); break; }
                const uint64_t L = std::min(B::kRows, len_of[c] - o);
                unsigned char* ob = bn.out[k];
                cudaError_t ce = cudaSuccess;
                ce = cudaMemcpyAsync(ob, w.dist + o, 8 * L, cudaMemcpyDeviceToHost, s.d2h);
                if (ce == cudaSuccess) ce = cudaMemcpyAsync(ob + 8 * B::kRows, w.cp + 3 * o, 24 * L, cudaMemcpyDeviceToHost, s.d2h);
                if (ce == cudaSuccess) ce = cudaMemcpyAsync(ob + 32 * B::kRows, w.face + o, 4 * L, cudaMemcpyDeviceToHost, s.d2h);
                if (ce == cudaSuccess) ce = cudaMemcpyAsync(ob + 36 * B::kRows, w.site + o, 4 * L, cudaMemcpyDeviceToHost, s.d2h);
                if (ce == cudaSuccess && flags) ce = cudaMemcpyAsync(ob + 40 * B::kRows, w.flags + o, 4 * L, cudaMemcpyDeviceToHost, s.d2h);
                if (ce == cudaSuccess) ce = cudaEventRecord(bn.out_ev[k], s.d2h);
                if (ce != cudaSuccess) { set_err(std::string("bounce D2H: ") + cudaGetErrorString(ce)); fail(P2M_ERR_CUDA); break; }
                pend[k] = Pend{start[c] + o, L, true};
            }
            if (rc == P2M_OK && cudaEventRecord(s.cev[3 * c + 2], s.d2h) != cudaSuccess) { set_err("d2h record"); fail(P2M_ERR_CUDA); }
            std::lock_guard<std::mutex> lk(mu);
            drained = c + 1;
            cv.notify_all();
        }
        for (int k = 0; k < B::kOut && rc == P2M_OK; ++k) {
            int r2 = unpack((int)((j + k) % B::kOut));
            if (r2 != P2M_OK) fail(r2);
        }
        std::lock_guard<std::mutex> lk(mu);
        if (rc != P2M_OK) out_rc = rc;
        drained = nch;
        cv.notify_all();
    });
    int rc = P2M_OK;
    uint64_t i = 0;
    for (size_t c = 0; c < nch && rc == P2M_OK; ++c) {
        const uint64_t len = len_of[c];
        const int k = (int)(c % Slot::kPipe);
        cudaStream_t st = s.pipe[k];
        Slot::Ws& w = s.ws[k];
        if (c >= (size_t)Slot::kPipe) {
            // staging set k is reused: its previous chunk's D2H copies must be enqueued (host side)
            // before this chunk's H2D may be ordered after them
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return drained >= c - Slot::kPipe + 1 || out_rc != P2M_OK; });
            if (out_rc != P2M_OK) break;
            lk.unlock();
            if (cudaStreamWaitEvent(s.h2d, s.cev[3 * (c - Slot::kPipe) + 1], 0) != cudaSuccess) { rc = P2M_ERR_CUDA; break; }
        }
        for (uint64_t o = 0; o < len; o += B::kRows, ++i) {
            const int kk = (int)(i % B::kIn);
            if (i >= (uint64_t)B::kIn && cudaEventSynchronize(bn.in_ev[kk]) != cudaSuccess) { set_err("bounce H2D failed"); rc = P2M_ERR_CUDA; break; }
            const uint64_t L = std::min(B::kRows, len - o);
            const CopyPool::Seg seg{bn.in[kk], q + 3 * (b + start[c] + o), 24 * L};
            bn.pack->run(&seg, 1);
            if (cudaMemcpyAsync(w.q + 3 * o, bn.in[kk], 24 * L, cudaMemcpyHostToDevice, s.h2d) != cudaSuccess ||
                cudaEventRecord(bn.in_ev[kk], s.h2d) != cudaSuccess) { set_err("bounce H2D enqueue failed"); rc = P2M_ERR_CUDA; break; }
        }
        if (rc != P2M_OK) break;
        cudaEvent_t ev_in = s.cev[3 * c], ev_k = s.cev[3 * c + 1];
        if (cudaEventRecord(ev_in, s.h2d) != cudaSuccess || cudaStreamWaitEvent(st, ev_in, 0) != cudaSuccess) { rc = P2M_ERR_CUDA; break; }
        if (serial_kernels && c > 0 && cudaStreamWaitEvent(st, s.cev[3 * (c - 1) + 1], 0) != cudaSuccess) { rc = P2M_ERR_CUDA; break; }
        if (c >= (size_t)Slot::kPipe && cudaStreamWaitEvent(st, s.cev[3 * (c - Slot::kPipe) + 2], 0) != cudaSuccess) { rc = P2M_ERR_CUDA; break; }
        p2m::dev::Out o{w.dist, w.cp, w.face, w.site, w.flags, nullptr, cnt ? s.agg : nullptr};
        rc = run_pipeline(e, s, w.q, len, o, cnt != nullptr, st, false, nullptr, false, &w.sc, k);
        if (rc != P2M_OK) break;
        if (cudaEventRecord(ev_k, st) != cudaSuccess) { rc = P2M_ERR_CUDA; break; }
        std::lock_guard<std::mutex> lk(mu);
        launched = c + 1;
        cv.notify_all();
    }
    if (rc != P2M_OK) {
        std::lock_guard<std::mutex> lk(mu);
        if (out_rc == P2M_OK) out_rc = rc;
        cv.notify_all();
    }
    out.join();
    if (rc == P2M_OK && out_rc != P2M_OK) { set_err(out_err); rc = out_rc; }
    if (rc != P2M_OK) return rc;
    CK(cudaStreamSynchronize(s.d2h));
    for (auto& st : s.pipe) CK(cudaStreamSynchronize(st));
    unsigned long long h[8] = {0};
    if (cnt) CK(cudaMemcpy(h, s.agg, sizeof h, cudaMemcpyDeviceToHost));
    uint64_t m = 0;
    for (uint64_t l : len_of) m += l;
    part.n_queries = m;
    part.candidates_visited = h[0];
    part.exact_evaluations = h[1];
    part.pruned = h[0] - h[1];
    part.kd_nodes_visited = h[2];
    part.filter_passes = h[4];
    part.warp_rare_iters = h[5];
    part.structure_bytes = h[6];
    part.scan_tiles = h[7];
    part.fallbacks = h[3];
    return P2M_OK;
}

P2M_API int p2m_query(p2m_engine* e, const double* q, uint64_t n, double* dist, double* cp, uint32_t* face,
                      uint32_t* site, uint32_t* flags, p2m_counters* cnt) {
    if (!e) { set_err("p2m_query: engine not built"); return P2M_ERR_NOT_BUILT; }
    if (n && (!q || !dist || !cp || !face || !site)) { set_err("p2m_query: null buffer"); return P2M_ERR_INVALID; }
    if (cnt) std::memset(cnt, 0, sizeof *cnt);
    if (!n) return P2M_OK;
    const int G = (int)e->slots.size();
    std::vector<int> rcs(G, P2M_OK);
    std::vector<p2m_counters> parts(G);
    std::vector<std::string> errs(G);
    auto work = [&](int g) {
        const uint64_t b = n * (uint64_t)g / G, en = n * (uint64_t)(g + 1) / G, m = en - b;
        parts[g] = p2m_counters{};
        if (!m) return;
        Slot& s = *e->slots[g];
        std::lock_guard<std::mutex> lk(s.mu);
        auto run = [&]() -> int {
            CK(cudaSetDevice(s.dev));
            // Host-buffer pipeline.  PCIe, not the kernels, bounds this path (24 B in + 44 B out per
            // row against ~1.6 G rows/s of kernels), so the schedule keeps both DMA directions busy:
            //  * copies are issued in row order on ONE stream per direction, so each copy runs at full
            //    link bandwidth instead of sharing it with the copies of later chunks;
            //  * chunks grow geometrically from ~m/32 rows, so the first results start leaving the GPU
            //    after a small H2D + kernel latency and the D2H stream then stays busy to the end;
            //  * kernels of chunk c run on compute stream c % kPipe with staging set c % kPipe, after
            //    its input landed and after the D2H of the chunk that used the set before it.
            std::vector<uint64_t> len_of;
            // big chunks each fill the GPU: their kernels run in chunk order (a later chunk whose input
            // landed early otherwise interleaves with an earlier one, which then finishes -- and starts
            // its D2H -- late: 291 vs 334 ms on c5 at 80/20, seen run to run)
            bool serial_kernels = false;
            if (e->e2e_chunks > 0) {
                const uint64_t k = (uint64_t)e->e2e_chunks;
                const uint64_t c0 = std::max<uint64_t>(1ull << 16, (m + k - 1) / k);
                for (uint64_t off = 0; off < m; off += c0) len_of.push_back(std::min(c0, m - off));
            } else if (!e->e2e_sched_set && m < 128ull * e->n_sites && m >= (1ull << 22)) {
                // Sparse batch (few rows per site, the regime of the warp tiles): a tile's cost is
                // nearly independent of its rows, so every extra chunk re-pays the lists -- c5 at
                // 100 M rows runs at 0.49 G rows/s whole, 0.42 in halves, 0.26 in eighths.  Few big
                // chunks, then, the last one smaller so that the drain (its D2H) is short: two equal
                // chunks and a tail (P2M_E2E_TAIL, default 0.1), kernels of consecutive chunks in
                // order (serial_kernels below).  Measured (100 M rows, pinned), c5: 358 ms geometric,
                // 302 in two halves, 292 at 45/45/10, 302 at 40/40/20; c4 (kernels as fast as the
                // copies): 199 geometric, 175 in halves, 167 at 45/45/10, 161 at 40/40/20.
                const uint64_t mt = std::max<uint64_t>(1ull << 18, (uint64_t)(e->e2e_sparse_tail * (double)m));
                if (mt < m) {
                    const uint64_t h0 = (m - mt + 1) / 2;
                    len_of.push_back(h0);
                    if (m - mt - h0) len_of.push_back(m - mt - h0);
                    len_of.push_back(mt);
                } else {
                    len_of.push_back(m);
                }
                serial_kernels = true;
            } else {
                // geometric: first chunk m*first, growing by `growth` up to m*cap, the last m*tail rows
                // as a separate small chunk (its D2H is the pipeline's drain)
                const double first = e->e2e_sched[0], growth = e->e2e_sched[1], cap = e->e2e_sched[2],
                             tail = e->e2e_sched[3];
                const uint64_t cmax = std::max<uint64_t>(1ull << 18, (uint64_t)(cap * (double)m));
                const uint64_t mt = std::min<uint64_t>(m, (uint64_t)(tail * (double)m));
                uint64_t cur = std::min(cmax, std::max<uint64_t>(1ull << 18, (uint64_t)(first * (double)m)));
                for (uint64_t off = 0; off < m - mt;) {
                    const uint64_t l = std::min(cur, m - mt - off);
                    len_of.push_back(l);
                    off += l;
                    cur = std::min(cmax, (uint64_t)(growth * (double)cur));
                }
                if (mt) len_of.push_back(mt);
            }
            if (len_of.size() > (size_t)Slot::kMaxChunks) {  // fold the tail into equal chunks
                const uint64_t c0 = (m + Slot::kMaxChunks - 1) / Slot::kMaxChunks;
                len_of.clear();
                for (uint64_t off = 0; off < m; off += c0) len_of.push_back(std::min(c0, m - off));
            }
            uint64_t maxlen = 0;
            for (uint64_t l : len_of) maxlen = std::max(maxlen, l);
            int rc = ensure_ws(s, maxlen, e->n_sites, (int)len_of.size());
            if (rc != P2M_OK) return rc;
            if (cnt) {
                CK(cudaMemsetAsync(s.agg, 0, sizeof(unsigned long long) * 8, s.pipe[0]));
                CK(cudaEventRecord(s.agg_ready, s.pipe[0]));
                for (int k = 1; k < Slot::kPipe; ++k) CK(cudaStreamWaitEvent(s.pipe[k], s.agg_ready, 0));
            }
            if (s.t0) CK(cudaEventRecord(s.t0, s.h2d));
            const bool bounce = !(host_pinned(q + 3 * b) && host_pinned(dist + b) && host_pinned(cp + 3 * b) &&
                                  host_pinned(face + b) && host_pinned(site + b) && (!flags || host_pinned(flags + b)));
            if (bounce) {
                rc = ensure_bounce(s);
                if (rc != P2M_OK) return rc;
                return run_bounce(e, s, q, dist, cp, face, site, flags, b, len_of, cnt, parts[g], serial_kernels);
            }
            uint64_t off = 0;
            for (size_t c = 0; c < len_of.size(); ++c) {
                const uint64_t len = len_of[c], r0 = b + off;
                off += len;
                const int k = (int)(c % Slot::kPipe);
                cudaStream_t st = s.pipe[k];
                Slot::Ws& w = s.ws[k];
                cudaEvent_t ev_in = s.cev[3 * c], ev_k = s.cev[3 * c + 1], ev_out = s.cev[3 * c + 2];
                if (c >= (size_t)Slot::kPipe) CK(cudaStreamWaitEvent(s.h2d, s.cev[3 * (c - Slot::kPipe) + 1], 0));
                CK(cudaMemcpyAsync(w.q, q + 3 * r0, 24 * len, cudaMemcpyHostToDevice, s.h2d));
                CK(cudaEventRecord(ev_in, s.h2d));
                CK(cudaStreamWaitEvent(st, ev_in, 0));
                if (serial_kernels && c > 0) CK(cudaStreamWaitEvent(st, s.cev[3 * (c - 1) + 1], 0));
                if (c >= (size_t)Slot::kPipe) CK(cudaStreamWaitEvent(st, s.cev[3 * (c - Slot::kPipe) + 2], 0));
                p2m::dev::Out o{w.dist, w.cp, w.face, w.site, w.flags, nullptr, cnt ? s.agg : nullptr};
                rc = run_pipeline(e, s, w.q, len, o, cnt != nullptr, st, false, nullptr, false, &w.sc, k);
                if (rc != P2M_OK) return rc;
                CK(cudaEventRecord(ev_k, st));
                CK(cudaStreamWaitEvent(s.d2h, ev_k, 0));
                CK(cudaMemcpyAsync(dist + r0, w.dist, 8 * len, cudaMemcpyDeviceToHost, s.d2h));
                CK(cudaMemcpyAsync(cp + 3 * r0, w.cp, 24 * len, cudaMemcpyDeviceToHost, s.d2h));
                CK(cudaMemcpyAsync(face + r0, w.face, 4 * len, cudaMemcpyDeviceToHost, s.d2h));
                CK(cudaMemcpyAsync(site + r0, w.site, 4 * len, cudaMemcpyDeviceToHost, s.d2h));
                if (flags) CK(cudaMemcpyAsync(flags + r0, w.flags, 4 * len, cudaMemcpyDeviceToHost, s.d2h));
                CK(cudaEventRecord(ev_out, s.d2h));
            }
            CK(cudaStreamSynchronize(s.d2h));
            if (s.t0) {
                for (size_t c = 0; c < len_of.size(); ++c) {
                    float a = 0, k = 0, o = 0;
                    cudaEventElapsedTime(&a, s.t0, s.cev[3 * c]);
                    cudaEventElapsedTime(&k, s.t0, s.cev[3 * c + 1]);
                    cudaEventElapsedTime(&o, s.t0, s.cev[3 * c + 2]);
                    std::fprintf(stderr, "e2e chunk %zu rows %llu: in %.3f  kernels %.3f  out %.3f ms\n", c,
                                 (unsigned long long)len_of[c], a, k, o);
                }
            }
            for (auto& st : s.pipe) CK(cudaStreamSynchronize(st));
            unsigned long long h[8] = {0};
            if (cnt) CK(cudaMemcpy(h, s.agg, sizeof h, cudaMemcpyDeviceToHost));
            parts[g].n_queries = m;
            parts[g].candidates_visited = h[0];
            parts[g].exact_evaluations = h[1];
            parts[g].pruned = h[0] - h[1];
            parts[g].kd_nodes_visited = h[2];
            parts[g].filter_passes = h[4];
            parts[g].warp_rare_iters = h[5];
            parts[g].structure_bytes = h[6];
            parts[g].scan_tiles = h[7];
            parts[g].fallbacks = h[3];
            return P2M_OK;
        };
        rcs[g] = run();
        if (rcs[g] != P2M_OK) errs[g] = p2m_last_error();
    };
    if (G == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int g = 0; g < G; ++g) th.emplace_back(work, g);
        for (auto& t : th) t.join();
    }
    for (int g = 0; g < G; ++g)
        if (rcs[g] != P2M_OK) { set_err(errs[g]); return rcs[g]; }
    if (cnt) {
        for (auto& c : parts) {
            cnt->n_queries += c.n_queries;
            cnt->candidates_visited += c.candidates_visited;
            cnt->exact_evaluations += c.exact_evaluations;
            cnt->pruned += c.pruned;
            cnt->kd_nodes_visited += c.kd_nodes_visited;
            cnt->filter_passes += c.filter_passes;
            cnt->warp_rare_iters += c.warp_rare_iters;
            cnt->structure_bytes += c.structure_bytes;
            cnt->scan_tiles += c.scan_tiles;
            cnt->fallbacks += c.fallbacks;
        }
    }
    return P2M_OK;
}

P2M_API int p2m_set_profiling(p2m_engine* e, int enable) {
    if (!e) { set_err("engine not built"); return P2M_ERR_NOT_BUILT; }
    e->profiling = enable != 0;
    for (auto& s : e->slots) s->recorded = 0;
    return P2M_OK;
}

// Mean per-call split over the calls recorded since profiling was (re)enabled; resets the ring.
P2M_API int p2m_last_timings(p2m_engine* e, int slot, float* ms) {
    if (!e || !ms || slot < 0 || slot >= (int)e->slots.size()) { set_err("p2m_last_timings: bad argument"); return P2M_ERR_INVALID; }
    Slot& s = *e->slots[slot];
    double acc[Slot::kEv] = {0};
    CK(cudaSetDevice(s.dev));
    const int nrec = std::min(s.recorded.load(), (int)Slot::kRing);
    for (int r = 0; r < nrec; ++r) {
        cudaEvent_t* ev = &s.ev[Slot::kEv * r];
        CK(cudaEventSynchronize(ev[Slot::kEv - 1]));
        float m;
        for (int k = 0; k + 1 < Slot::kEv; ++k) { CK(cudaEventElapsedTime(&m, ev[k], ev[k + 1])); acc[k] += m; }
        CK(cudaEventElapsedTime(&m, ev[0], ev[Slot::kEv - 1])); acc[Slot::kEv - 1] += m;
    }
    for (int k = 0; k < Slot::kEv; ++k) ms[k] = nrec ? (float)(acc[k] / nrec) : 0.0f;
    s.recorded = 0;
    return P2M_OK;
}

P2M_API int p2m_set_scan_mode(p2m_engine* e, int mode) {
    if (!e) { set_err("engine not built"); return P2M_ERR_NOT_BUILT; }
    if (mode != P2M_SCAN_GROUPED && mode != P2M_SCAN_FUSED) { set_err("p2m_set_scan_mode: unknown mode"); return P2M_ERR_INVALID; }
    e->scan_mode = mode;
    return P2M_OK;
}

P2M_API int p2m_set_nns_strategy(p2m_engine* e, int strategy) {
    if (!e) { set_err("engine not built"); return P2M_ERR_NOT_BUILT; }
    if (strategy != P2M_NNS_GRID && strategy != P2M_NNS_KDTREE && strategy != P2M_NNS_WALK) {
        set_err("p2m_set_nns_strategy: unknown strategy");
        return P2M_ERR_INVALID;
    }
    if (strategy == P2M_NNS_WALK && !e->has_adj) {
        set_err("p2m_set_nns_strategy: DelaunayWalk needs the engine's Delaunay adjacency (desc.adj_offsets)");
        return P2M_ERR_INVALID;
    }
    for (auto& s : e->slots) {
        std::lock_guard<std::mutex> lk(s->pmu);
        s->params.nns = strategy;
    }
    return P2M_OK;
}

// Count the kernels one p2m_query_device call launches by capturing it into a CUDA graph.
P2M_API int p2m_kernels_per_query(p2m_engine* e, uint64_t n, int* launches) {
    if (!e || !launches) { set_err("p2m_kernels_per_query: bad argument"); return P2M_ERR_INVALID; }
    Slot& s = *e->slots[0];
    CK(cudaSetDevice(s.dev));
    if (!n) n = 1;
    double *q = nullptr, *dist = nullptr, *cp = nullptr;
    uint32_t *face = nullptr, *site = nullptr;
    CK(cudaMalloc(&q, 24 * n)); CK(cudaMemset(q, 0, 24 * n));
    CK(cudaMalloc(&dist, 8 * n)); CK(cudaMalloc(&cp, 24 * n)); CK(cudaMalloc(&face, 4 * n)); CK(cudaMalloc(&site, 4 * n));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    bool prof = e->profiling;
    e->profiling = false;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    p2m::dev::Out o{dist, cp, face, site, nullptr, nullptr, nullptr};
    int rc = run_pipeline(e, s, q, n, o, false, st, false, nullptr);
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(st, &g);
    e->profiling = prof;
    int k = 0;
    if (rc == P2M_OK && g) {
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(g, nodes.data(), &nn);
        for (auto& x : nodes) {
            cudaGraphNodeType t;
            cudaGraphNodeGetType(x, &t);
            if (t == cudaGraphNodeTypeKernel) ++k;
        }
    }
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(st);
    cudaFree(q); cudaFree(dist); cudaFree(cp); cudaFree(face); cudaFree(site);
    if (rc != P2M_OK) return rc;
    *launches = k;
    return P2M_OK;
}
