// p2m_grid.cu -- the exact cell-locate grid built on the device from the sites alone, for engines
// whose descriptor carries no Voronoi cell boxes (desc.site_cell_box == NULL: an external builder,
// INTEGRATION.md).  Same grid geometry and the same lookup as the host build from cell boxes
// (p2m_engine.cu build_grid, p2m_traverse.cuh nearest_site_cl), different candidate rule:
//
//   cell B with centre c and half-diagonal h; s0 = nearest site of c (exact k-d descent), d0 = |c - s0|.
//   (1) every site nearest to some q in B lies within d0 + 2h of c:
//         |q - s*| <= |q - s0| <= h + d0   and   |s* - c| <= |s* - q| + |q - c| <= d0 + 2h;
//   (2) it also satisfies |q - s| <= |q - t| at that q for every other site t -- in particular for
//       t = s0: f(q) = |q - s|^2 - |q - s0|^2 is affine in q, so its minimum over B is attained at a
//       corner, and a site whose corner minimum is > 0 can be nearest nowhere in B.
//   A cell lists every site passing (1) (k-d radius search) and (2) (8 corners, with a relative
//   tolerance so rounding only ever keeps a site): a superset of the sites whose closed Voronoi cell
//   meets B, hence the lookup's lexicographic (d^2, id) minimum is the exact nearest site with
//   lowest-id ties (REF/SPEC.md:482-487).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <vector>

#include "p2m_device.cuh"
#include "p2m_traverse.cuh"

namespace p2m {
namespace dev {

namespace {

struct GridGeom {
    double lo[3], inv[3];
    uint32_t res[3];
};

// Visit every k-d node within radius sqrt(r2) of c (explicit stack; the tree is left-balanced, depth
// <= 33), calling emit(id, site xyz) for each.
template <class Emit>
__device__ __forceinline__ void radius_search(const Params& p, V c, double r2, Emit&& emit) {
    int stack[64];
    int sp = 0;
    stack[sp++] = 0;
    const int N = (int)p.n_nodes;
    while (sp) {
        const int k = stack[--sp];
        if (k >= N) continue;
        const D4 nd = ldg4(p.kd + k);
        const uint64_t meta = (uint64_t)__double_as_longlong(nd.w);
        const V s{nd.x, nd.y, nd.z};
        if (vd2(c, s) <= r2) emit((uint32_t)(meta & kIdMask), s);
        const int dim = (int)((meta >> kDimShift) & 3);
        const double diff = (dim == 0 ? c.x : (dim == 1 ? c.y : c.z)) - (dim == 0 ? nd.x : (dim == 1 ? nd.y : nd.z));
        const int right = diff > 0.0;
        const int close_c = 2 * k + 1 + right, far_c = 2 * k + 2 - right;
        if (diff * diff <= r2 && sp < 64) stack[sp++] = far_c;
        if (sp < 64) stack[sp++] = close_c;
    }
}

template <bool kFill>
__global__ void __launch_bounds__(128) k_grid_cells(Params p, GridGeom g, uint64_t ncell, uint32_t* __restrict__ cnt,
                                                    const uint32_t* __restrict__ off, uint32_t* __restrict__ out) {
    const uint64_t cell = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= ncell) return;
    const uint32_t ix = (uint32_t)(cell % g.res[0]), iy = (uint32_t)((cell / g.res[0]) % g.res[1]),
                   iz = (uint32_t)(cell / ((uint64_t)g.res[0] * g.res[1]));
    double lo[3], hi[3];
    const uint32_t ii[3] = {ix, iy, iz};
    for (int k = 0; k < 3; ++k) {
        // the cell's box, widened by a relative margin: q maps to this cell only if q lies in it
        const double w = 1.0 / g.inv[k];
        lo[k] = g.lo[k] + (double)ii[k] * w;
        hi[k] = g.lo[k] + (double)(ii[k] + 1) * w;
        const double m = 1e-9 * (fabs(lo[k]) + fabs(hi[k]) + w);
        lo[k] -= m;
        hi[k] += m;
    }
    const V c{0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    const double h = 0.5 * sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                                (hi[2] - lo[2]) * (hi[2] - lo[2]));
    const NN n0 = nearest_site(p, c);
    // the position of s0: re-found by a radius search of radius d0 (the same fp64 d^2 as the descent)
    const double d0 = sqrt(n0.d2);
    const double R = (d0 + 2.0 * h) * (1.0 + 1e-9) + 1e-300;
    V p0{0, 0, 0};
    radius_search(p, c, n0.d2 * (1.0 + 1e-12), [&](uint32_t id, V s) { if (id == n0.id) p0 = s; });
    uint32_t n = 0;
    const uint32_t base = kFill ? off[cell] : 0u;
    radius_search(p, c, R * R, [&](uint32_t id, V s) {
        // affine test against s0 at the 8 corners (keep if some corner is not strictly closer to s0)
        bool keep = id == n0.id;
        for (int corner = 0; corner < 8 && !keep; ++corner) {
            const V q{(corner & 1) ? hi[0] : lo[0], (corner & 2) ? hi[1] : lo[1], (corner & 4) ? hi[2] : lo[2]};
            const double a = vd2(q, s), b = vd2(q, p0);
            if (a - b <= 1e-9 * (a + b)) keep = true;
        }
        if (!keep) return;
        if (kFill) out[base + n] = id;
        ++n;
    });
    if (!kFill) cnt[cell] = n;
}

}  // namespace

// Device build of the cell-locate grid over kd (S nodes, the packed k-d tree) on device `dev`.
// Fills off[ncell+1] and site[] on the host; returns false (and leaves them empty) on failure or if
// the grid would exceed 2^32 pairs.
bool build_grid_device(int dev, const D4* kd_host, uint32_t S, const double lo[3], const double inv[3],
                       const uint32_t res[3], std::vector<uint32_t>& off, std::vector<uint32_t>& site) {
    off.clear();
    site.clear();
    if (cudaSetDevice(dev) != cudaSuccess) return false;
    const uint64_t ncell = (uint64_t)res[0] * res[1] * res[2];
    GridGeom g;
    for (int k = 0; k < 3; ++k) { g.lo[k] = lo[k]; g.inv[k] = inv[k]; g.res[k] = res[k]; }
    D4* kd = nullptr;
    uint32_t *cnt = nullptr, *o = nullptr, *out = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    bool ok = false;
    do {
        if (cudaMalloc(&kd, sizeof(D4) * S) != cudaSuccess) break;
        if (cudaMemcpy(kd, kd_host, sizeof(D4) * S, cudaMemcpyHostToDevice) != cudaSuccess) break;
        if (cudaMalloc(&cnt, 4 * (ncell + 1)) != cudaSuccess || cudaMalloc(&o, 4 * (ncell + 1)) != cudaSuccess) break;
        if (cudaMemset(cnt + ncell, 0, 4) != cudaSuccess) break;
        Params p{};
        p.kd = kd;
        p.n_nodes = S;
        const unsigned blocks = (unsigned)((ncell + 127) / 128);
        k_grid_cells<false><<<blocks, 128>>>(p, g, ncell, cnt, nullptr, nullptr);
        if (cudaGetLastError() != cudaSuccess) break;
        // pair count in 64 bits first (the u32 offsets must not overflow)
        std::vector<uint32_t> hc(ncell);
        if (cudaMemcpy(hc.data(), cnt, 4 * ncell, cudaMemcpyDeviceToHost) != cudaSuccess) break;
        uint64_t total = 0;
        for (uint32_t v : hc) total += v;
        if (total >= (1ull << 32)) break;
        if (cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, o, (int64_t)(ncell + 1)) != cudaSuccess) break;
        if (cudaMalloc(&tmp, tb) != cudaSuccess) break;
        if (cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, o, (int64_t)(ncell + 1)) != cudaSuccess) break;
        if (cudaMalloc(&out, 4 * (total ? total : 1)) != cudaSuccess) break;
        k_grid_cells<true><<<blocks, 128>>>(p, g, ncell, nullptr, o, out);
        if (cudaGetLastError() != cudaSuccess) break;
        off.resize(ncell + 1);
        site.resize(total);
        if (cudaMemcpy(off.data(), o, 4 * (ncell + 1), cudaMemcpyDeviceToHost) != cudaSuccess) break;
        if (total && cudaMemcpy(site.data(), out, 4 * total, cudaMemcpyDeviceToHost) != cudaSuccess) break;
        ok = true;
    } while (false);
    cudaFree(kd); cudaFree(cnt); cudaFree(o); cudaFree(out); cudaFree(tmp);
    if (!ok) { cudaGetLastError(); off.clear(); site.clear(); }
    return ok;
}

}  // namespace dev
}  // namespace p2m
