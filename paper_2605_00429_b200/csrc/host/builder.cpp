// builder.cpp -- host build phase: validate_mesh, build_bvh, make_bounded_site_set, augment_sites,
// cell corners, build_all_tables, per-face spheres (REF/SPEC.md:112-456).
#include "builder.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <unordered_map>
#include <unordered_set>

#include "util.hpp"
#include "voronoi.hpp"

namespace p2m {

uint64_t hash_mesh(const double* v, uint64_t nv, const uint32_t* f, uint64_t nf) {
    // FNV-1a over the raw little-endian bytes, folded through mix64
    uint64_t h = 0xcbf29ce484222325ull;
    auto eat = [&](const void* p, size_t n) {
        const unsigned char* c = (const unsigned char*)p;
        for (size_t i = 0; i < n; ++i) { h ^= c[i]; h *= 0x100000001b3ull; }
    };
    eat(&nv, 8); eat(&nf, 8);
    eat(v, nv * 24);
    eat(f, nf * 12);
    return mix64(h);
}

// validate_mesh (REF/SPEC.md:132-140, 151-157): exact-duplicate vertex merge (first occurrence
// wins, order preserved) and removal of zero-area faces (REF geom.cpp:76-80 criterion, plus the
// SPEC's area floor 1e-14 * diag^2).
static void validate(const double* v, uint64_t nv, const uint32_t* f, uint64_t nf, bool strict,
                     HostEngine& h) {
    if (nv == 0 || nf == 0) throw std::invalid_argument("validate_mesh: empty mesh");
    for (uint64_t i = 0; i < 3 * nf; ++i)
        if (f[i] >= nv) throw std::invalid_argument("validate_mesh: face index out of range");
    for (uint64_t i = 0; i < 3 * nv; ++i)
        if (!std::isfinite(v[i])) throw std::invalid_argument("validate_mesh: non-finite vertex");
    std::vector<uint32_t> order(nv);
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        for (int k = 0; k < 3; ++k) {
            double x = v[3 * (uint64_t)a + k], y = v[3 * (uint64_t)b + k];
            if (x != y) return x < y;
        }
        return a < b;
    });
    std::vector<uint32_t> canon(nv);
    for (uint64_t i = 0; i < nv; ++i) {
        uint32_t a = order[i];
        if (i > 0) {
            uint32_t p = order[i - 1];
            if (v[3 * (uint64_t)a] == v[3 * (uint64_t)p] && v[3 * (uint64_t)a + 1] == v[3 * (uint64_t)p + 1] &&
                v[3 * (uint64_t)a + 2] == v[3 * (uint64_t)p + 2]) {
                canon[a] = canon[p];
                continue;
            }
        }
        canon[a] = a;
    }
    std::vector<uint32_t> newid(nv, UINT32_MAX);
    h.V.clear();
    for (uint64_t i = 0; i < nv; ++i)
        if (canon[i] == i) {
            newid[i] = (uint32_t)(h.V.size() / 3);
            h.V.insert(h.V.end(), v + 3 * i, v + 3 * i + 3);
        }
    h.stats.merged_vertices = nv - h.V.size() / 3;
    Box b;
    for (uint64_t i = 0; i < nv; ++i) b.add(ld3(v + 3 * i));
    const double floor_area = 1e-14 * b.diag() * b.diag();
    h.F.clear();
    uint64_t removed = 0;
    for (uint64_t t = 0; t < nf; ++t) {
        uint32_t i0 = newid[canon[f[3 * t]]], i1 = newid[canon[f[3 * t + 1]]], i2 = newid[canon[f[3 * t + 2]]];
        V3 a = ld3(&h.V[3 * (uint64_t)i0]), bb = ld3(&h.V[3 * (uint64_t)i1]), c = ld3(&h.V[3 * (uint64_t)i2]);
        bool bad = i0 == i1 || i1 == i2 || i0 == i2 || tri_degenerate(a, bb, c) ||
                   0.5 * len(cross(bb - a, c - a)) < floor_area;
        if (bad) {
            if (strict) throw GeometryErr("validate_mesh: degenerate face (strict mode)");
            ++removed;
            continue;
        }
        h.F.push_back(i0); h.F.push_back(i1); h.F.push_back(i2);
    }
    if (h.F.empty()) throw GeometryErr("validate_mesh: all faces degenerate");
    h.stats.removed_faces = removed;
}

static double mean_edge(const HostEngine& h) {
    std::vector<uint64_t> e;
    e.reserve(h.F.size());
    for (size_t t = 0; t < h.F.size(); t += 3)
        for (int k = 0; k < 3; ++k) {
            uint32_t a = h.F[t + k], b = h.F[t + (k + 1) % 3];
            if (a > b) std::swap(a, b);
            e.push_back((uint64_t)a << 32 | b);
        }
    std::sort(e.begin(), e.end());
    e.erase(std::unique(e.begin(), e.end()), e.end());
    double s = 0.0;
    for (uint64_t k : e) {
        uint32_t a = (uint32_t)(k >> 32), b = (uint32_t)k;
        s += std::sqrt(d2(ld3(&h.V[3 * (uint64_t)a]), ld3(&h.V[3 * (uint64_t)b])));
    }
    return e.empty() ? 0.0 : s / (double)e.size();
}

// Derived per-face arrays: fp64 triangles and minimal bounding spheres.
static void face_arrays(HostEngine& h) {
    const uint64_t nf = h.F.size() / 3;
    h.tri.resize(9 * nf);
    h.sphere.resize(4 * nf);
    for (uint64_t t = 0; t < nf; ++t) {
        for (int k = 0; k < 3; ++k)
            for (int c = 0; c < 3; ++c) h.tri[9 * t + 3 * k + c] = h.V[3 * (uint64_t)h.F[3 * t + k] + c];
        tri_sphere(ld3(&h.tri[9 * t]), ld3(&h.tri[9 * t + 3]), ld3(&h.tri[9 * t + 6]), &h.sphere[4 * t]);
    }
}

static void build_adjacency(HostEngine& h, std::vector<std::vector<uint32_t>>& nbr);

static Box outer_box(const HostEngine& h) {
    // cube about D's centre that contains every sentinel-bounded cell (<= 2x the sentinel
    // half-extent along any axis for sites inside D); 3x for margin
    V3 c = h.sentinel_box.center();
    V3 e = h.sentinel_box.ext() * 0.5;
    double m = 3.0 * std::max({e.x, e.y, e.z});
    Box b;
    b.lo = c - V3{m, m, m};
    b.hi = c + V3{m, m, m};
    return b;
}

static constexpr int kKnn = 24;

void cell_corners(const HostEngine& h, uint32_t site, std::vector<V3>& out) {
    CellClipper cc(h.sites, h.tree, outer_box(h), h.sentinel_ids, 8, h.eps, kKnn);
    cc.compute(site, out, nullptr);
}

void delaunay_adjacency(const double* xyz, uint64_t n, int n_threads, std::vector<uint64_t>& off,
                        std::vector<uint32_t>& adj) {
    // the builder's bounded site set (REF/SPEC.md:247-255) around the points, cells by clipping
    HostEngine h;
    Box aabb;
    for (uint64_t i = 0; i < n; ++i) aabb.add(ld3(xyz + 3 * i));
    h.D = aabb.scaled(10.0, 0.1);
    h.sentinel_box = h.D.scaled(4.0, 0.0);
    h.eps = 1e-12 * h.D.diag();
    for (uint64_t i = 0; i < n; ++i) h.sites.push_back(ld3(xyz + 3 * i));
    for (int i = 0; i < 8; ++i) {
        h.sentinel_ids[i] = (uint32_t)h.sites.size();
        h.sites.push_back(V3{(i & 1) ? h.sentinel_box.hi.x : h.sentinel_box.lo.x,
                             (i & 2) ? h.sentinel_box.hi.y : h.sentinel_box.lo.y,
                             (i & 4) ? h.sentinel_box.hi.z : h.sentinel_box.lo.z});
    }
    h.tree.build(h.sites);
    const Box outer = outer_box(h);
    std::vector<std::vector<uint32_t>> nbr(n + 8);
    parallel_for(n, hw_threads(n_threads), 32, [&](uint64_t b, uint64_t e, int) {
        CellClipper cc(h.sites, h.tree, outer, h.sentinel_ids, 8, h.eps, kKnn);
        std::vector<V3> corners;
        for (uint64_t s = b; s < e; ++s) cc.compute((uint32_t)s, corners, &nbr[s]);
    });
    build_adjacency(h, nbr);
    // drop the sentinels: for q inside D = AABB x 10 a sentinel is never closer than the current
    // site of a walk that starts at a real site, so the walk never needs them
    off.assign(n + 1, 0);
    adj.clear();
    for (uint64_t s = 0; s < n; ++s) {
        for (uint64_t k = h.adj_off[s]; k < h.adj_off[s + 1]; ++k)
            if (h.adj[k] < n) adj.push_back(h.adj[k]);
        off[s + 1] = adj.size();
    }
}

void finish_engine(HostEngine& h) {
    h.site_xyz.resize(3 * h.sites.size());
    for (size_t i = 0; i < h.sites.size(); ++i) {
        h.site_xyz[3 * i] = h.sites[i].x; h.site_xyz[3 * i + 1] = h.sites[i].y; h.site_xyz[3 * i + 2] = h.sites[i].z;
    }
    h.tree.build(h.sites);
}

static void prep_mesh(const double* v, uint64_t nv, const uint32_t* f, uint64_t nf,
                      const p2m_build_config& cfg, HostEngine& h) {
    validate(v, nv, f, nf, cfg.strict_mesh != 0, h);
    h.mesh_hash = hash_mesh(h.V.data(), h.V.size() / 3, h.F.data(), h.F.size() / 3);
    h.stats.n_vertices = h.V.size() / 3;
    h.stats.n_faces = h.F.size() / 3;
    face_arrays(h);
    for (uint64_t i = 0; i < h.V.size() / 3; ++i) h.aabb.add(ld3(&h.V[3 * i]));
}

// Delaunay adjacency CSR: the union of both directions of every facet-neighbour relation (a facet
// dropped within the clipping tolerance on one side is still an edge), sorted per site.
static void build_adjacency(HostEngine& h, std::vector<std::vector<uint32_t>>& nbr) {
    const uint64_t S = nbr.size();
    // sentinel cells are never built: their mutual facets are added as a complete graph on the 8
    // sentinels (a supergraph of the Delaunay graph keeps the walk exact), their facets with real
    // sites come from the real sites' cells
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j)
            if (i != j && h.sentinel_ids[i] < S && h.sentinel_ids[j] < S) nbr[h.sentinel_ids[i]].push_back(h.sentinel_ids[j]);
    std::vector<uint64_t> cnt(S + 1, 0);
    for (uint64_t s = 0; s < S; ++s)
        for (uint32_t w : nbr[s]) { ++cnt[s + 1]; ++cnt[w + 1]; }
    for (uint64_t s = 0; s < S; ++s) cnt[s + 1] += cnt[s];
    std::vector<uint32_t> all(cnt[S]);
    std::vector<uint64_t> cur(cnt.begin(), cnt.end() - 1);
    for (uint64_t s = 0; s < S; ++s)
        for (uint32_t w : nbr[s]) { all[cur[s]++] = w; all[cur[w]++] = (uint32_t)s; }
    h.adj_off.assign(S + 1, 0);
    h.adj.clear();
    h.adj.reserve(all.size() / 2 + 16);
    for (uint64_t s = 0; s < S; ++s) {
        auto b = all.begin() + cnt[s], e = all.begin() + cnt[s + 1];
        std::sort(b, e);
        e = std::unique(b, e);
        for (auto it = b; it != e; ++it)
            if (*it != s) h.adj.push_back(*it);
        h.adj_off[s + 1] = h.adj.size();
        std::vector<uint32_t>().swap(nbr[s]);
    }
}

// Flatten the per-site balls and the BVH into a p2m_table_job and run the delegated executor.
static void run_table_job(HostEngine& h, std::vector<std::vector<Ball>>& site_balls, p2m_table_fn fn,
                          void* ctx) {
    const uint64_t S = site_balls.size();
    std::vector<uint64_t> boff(S + 1, 0);
    for (uint64_t s = 0; s < S; ++s) boff[s + 1] = boff[s] + site_balls[s].size();
    std::vector<double> balls(4 * boff[S]);
    for (uint64_t s = 0; s < S; ++s) {
        double* o = &balls[4 * boff[s]];
        for (const Ball& b : site_balls[s]) { o[0] = b.c.x; o[1] = b.c.y; o[2] = b.c.z; o[3] = b.r2; o += 4; }
        std::vector<Ball>().swap(site_balls[s]);
    }
    const auto& nodes = h.bvh.nodes();
    std::vector<double> nbox(6 * nodes.size());
    std::vector<uint32_t> nmeta(3 * nodes.size());
    for (size_t i = 0; i < nodes.size(); ++i) {
        const BvhNode& n = nodes[i];
        double* b = &nbox[6 * i];
        b[0] = n.box.lo.x; b[1] = n.box.lo.y; b[2] = n.box.lo.z; b[3] = n.box.hi.x; b[4] = n.box.hi.y; b[5] = n.box.hi.z;
        nmeta[3 * i] = n.right; nmeta[3 * i + 1] = n.first; nmeta[3 * i + 2] = n.count;
    }
    p2m_table_job job{};
    job.n_sites = S;
    job.ball_off = boff.data();
    job.balls = balls.data();
    job.n_faces = h.tri.size() / 9;
    job.tri = h.tri.data();
    job.n_nodes = nodes.size();
    job.node_box = nbox.data();
    job.node_meta = nmeta.data();
    job.perm = h.bvh.perm().data();
    uint32_t* lists = nullptr;
    const int rc = fn(ctx, &job, h.off.data(), &lists);
    if (rc != 0) {
        std::free(lists);
        throw std::runtime_error(std::string("build_all_tables: table executor failed (") + std::to_string(rc) + "): " + get_error());
    }
    if (h.off[0] != 0) { std::free(lists); throw std::runtime_error("build_all_tables: bad offsets from executor"); }
    for (uint64_t s = 0; s < S; ++s)
        if (h.off[s + 1] < h.off[s]) { std::free(lists); throw std::runtime_error("build_all_tables: bad offsets from executor"); }
    h.lists.assign(lists, lists + h.off[S]);
    std::free(lists);
}

std::unique_ptr<HostEngine> build_engine_mesh_only(const double* v, uint64_t nv, const uint32_t* f,
                                                   uint64_t nf, const p2m_build_config& cfg) {
    auto hp = std::make_unique<HostEngine>();
    hp->cfg = cfg;
    prep_mesh(v, nv, f, nf, cfg, *hp);
    return hp;
}

std::unique_ptr<HostEngine> build_engine(const double* v, uint64_t nv, const uint32_t* f, uint64_t nf,
                                         const p2m_build_config& cfg, p2m_table_fn table_fn,
                                         void* table_ctx) {
    Timer total;
    auto hp = std::make_unique<HostEngine>();
    HostEngine& h = *hp;
    h.cfg = cfg;
    h.stats.n_input_vertices = nv;
    h.stats.n_input_faces = nf;
    if (!(cfg.alpha > 0) || cfg.k < 1 || !(cfg.rho > 0) || cfg.max_rounds < 1 || !(cfg.domain_scale >= 1.0))
        throw std::invalid_argument("build: invalid config (alpha>0, k>=1, rho>0, rounds>=1, domain_scale>=1)");
    prep_mesh(v, nv, f, nf, cfg, h);
    const uint64_t NV = h.V.size() / 3, NF = h.F.size() / 3;
    h.bvh.build(h.tri.data(), NF, 4);
    h.stats.mean_edge = mean_edge(h);
    // make_bounded_site_set (REF/SPEC.md:247-255): D = AABB x domain_scale, sentinels at the
    // corners of D scaled 4x.  Flat axes of D are padded to 10% of the largest extent.
    h.D = h.aabb.scaled(cfg.domain_scale, 0.1);
    h.sentinel_box = h.D.scaled(4.0, 0.0);
    h.eps = 1e-12 * h.D.diag();
    h.sites.clear();
    h.kind.clear();
    for (uint64_t i = 0; i < NV; ++i) { h.sites.push_back(ld3(&h.V[3 * i])); h.kind.push_back(P2M_SITE_MESH_VERTEX); }
    for (int i = 0; i < 8; ++i) {
        V3 c{(i & 1) ? h.sentinel_box.hi.x : h.sentinel_box.lo.x, (i & 2) ? h.sentinel_box.hi.y : h.sentinel_box.lo.y,
             (i & 4) ? h.sentinel_box.hi.z : h.sentinel_box.lo.z};
        h.sentinel_ids[i] = (uint32_t)h.sites.size();
        h.sites.push_back(c);
        h.kind.push_back(P2M_SITE_SENTINEL);
    }
    h.refs.assign(3 * h.sites.size(), std::nan(""));
    const int threads = hw_threads(cfg.n_threads);
    const double tau = cfg.alpha * h.stats.mean_edge;
    h.stats.tau = tau;
    const Box outer = outer_box(h);
    h.tree.build(h.sites);

    // ---- augment_sites (REF/SPEC.md:350-358) ----
    Timer t_aug;
    double t_vor = 0.0;
    int rounds_used = 0;
    std::vector<V3> accepted_aux;  // for the tau/4 dedup rule (REF/SPEC.md:369)
    if (cfg.augment && tau > 0.0) {
        for (int round = 0; round < cfg.max_rounds; ++round) {
            Timer tv;
            // grid_density_map over Voronoi vertices inside D (REF/SPEC.md:323-331).  A corner
            // shared by m cells is counted m/4 times (4 = cells per corner in general position), so
            // degenerate vertices where many cells meet weigh as the circumcentre clusters they
            // stand for.
            std::vector<std::vector<uint64_t>> keys(threads);
            const uint64_t S = h.sites.size();
            parallel_for(S, threads, 64, [&](uint64_t b, uint64_t e, int w) {
                CellClipper cc(h.sites, h.tree, outer, h.sentinel_ids, 8, h.eps, kKnn);
                std::vector<V3> corners;
                for (uint64_t s = b; s < e; ++s) {
                    if (h.kind[s] == P2M_SITE_SENTINEL) continue;
                    cc.compute((uint32_t)s, corners, nullptr);
                    for (const V3& u : corners) {
                        if (!h.D.contains(u)) continue;
                        uint64_t ix = (uint64_t)std::floor((u.x - h.D.lo.x) / tau);
                        uint64_t iy = (uint64_t)std::floor((u.y - h.D.lo.y) / tau);
                        uint64_t iz = (uint64_t)std::floor((u.z - h.D.lo.z) / tau);
                        keys[w].push_back((ix & 0x1FFFFF) << 42 | (iy & 0x1FFFFF) << 21 | (iz & 0x1FFFFF));
                    }
                }
            });
            t_vor += tv.s();
            std::vector<uint64_t> all;
            for (auto& k : keys) all.insert(all.end(), k.begin(), k.end());
            std::sort(all.begin(), all.end());
            // flag_dense_cells (REF/SPEC.md:332-340): count >= k, by count desc then key asc
            std::vector<std::pair<uint64_t, uint64_t>> dense;  // (-count via ~, key)
            for (size_t i = 0; i < all.size();) {
                size_t j = i;
                while (j < all.size() && all[j] == all[i]) ++j;
                double cnt = (double)(j - i) / 4.0;
                if (cnt >= (double)cfg.k) dense.push_back({(uint64_t)(j - i), all[i]});
                i = j;
            }
            std::sort(dense.begin(), dense.end(), [](auto& a, auto& b) {
                return a.first > b.first || (a.first == b.first && a.second < b.second);
            });
            if (dense.empty()) break;
            // make_auxiliary_cluster (REF/SPEC.md:341-349): centre + 14-direction ring at rho*tau
            const double inv3 = 1.0 / std::sqrt(3.0);
            const V3 dirs[14] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1},
                                 {-inv3, -inv3, -inv3}, {inv3, -inv3, -inv3}, {-inv3, inv3, -inv3},
                                 {inv3, inv3, -inv3}, {-inv3, -inv3, inv3}, {inv3, -inv3, inv3},
                                 {-inv3, inv3, inv3}, {inv3, inv3, inv3}};
            const double q = tau / 4.0, q2 = q * q;
            std::unordered_map<uint64_t, std::vector<uint32_t>> grid;  // accepted aux, cell size tau/4
            auto gkey = [&](V3 p, int dx, int dy, int dz) {
                int64_t ix = (int64_t)std::floor((p.x - h.D.lo.x) / q) + dx;
                int64_t iy = (int64_t)std::floor((p.y - h.D.lo.y) / q) + dy;
                int64_t iz = (int64_t)std::floor((p.z - h.D.lo.z) / q) + dz;
                return (uint64_t)(ix & 0x1FFFFF) << 42 | (uint64_t)(iy & 0x1FFFFF) << 21 | (uint64_t)(iz & 0x1FFFFF);
            };
            for (uint32_t i = 0; i < accepted_aux.size(); ++i) grid[gkey(accepted_aux[i], 0, 0, 0)].push_back(i);
            std::vector<V3> fresh;
            for (auto& dc : dense) {
                uint64_t key = dc.second;
                V3 cen{h.D.lo.x + ((double)(key >> 42 & 0x1FFFFF) + 0.5) * tau,
                       h.D.lo.y + ((double)(key >> 21 & 0x1FFFFF) + 0.5) * tau,
                       h.D.lo.z + ((double)(key & 0x1FFFFF) + 0.5) * tau};
                for (int r = 0; r < 15; ++r) {
                    V3 p = r == 0 ? cen : cen + dirs[r - 1] * (cfg.rho * tau);
                    bool drop = false;
                    for (int dx = -1; dx <= 1 && !drop; ++dx)
                        for (int dy = -1; dy <= 1 && !drop; ++dy)
                            for (int dz = -1; dz <= 1 && !drop; ++dz) {
                                auto it = grid.find(gkey(p, dx, dy, dz));
                                if (it == grid.end()) continue;
                                for (uint32_t j : it->second)
                                    if (d2(p, accepted_aux[j]) <= q2) { drop = true; break; }
                            }
                    if (!drop) {
                        double dd;  // exact coincidence with an existing site (REF/SPEC.md:344)
                        uint32_t w = h.tree.nearest(p, INFINITY, &dd);
                        if (w != UINT32_MAX && dd == 0.0) drop = true;
                    }
                    if (drop) continue;
                    grid[gkey(p, 0, 0, 0)].push_back((uint32_t)accepted_aux.size());
                    accepted_aux.push_back(p);
                    fresh.push_back(p);
                }
            }
            if (fresh.empty()) break;
            ++rounds_used;
            // projection of every auxiliary site onto the mesh (bvh_closest_point)
            const size_t base = h.sites.size();
            h.sites.insert(h.sites.end(), fresh.begin(), fresh.end());
            h.kind.insert(h.kind.end(), fresh.size(), (uint8_t)P2M_SITE_AUXILIARY);
            h.refs.resize(3 * h.sites.size(), std::nan(""));
            parallel_for(fresh.size(), threads, 256, [&](uint64_t b, uint64_t e, int) {
                for (uint64_t i = b; i < e; ++i) {
                    double dd;
                    V3 p;
                    h.bvh.closest(fresh[i], &dd, &p);
                    h.refs[3 * (base + i)] = p.x; h.refs[3 * (base + i) + 1] = p.y; h.refs[3 * (base + i) + 2] = p.z;
                }
            });
            h.tree.build(h.sites);
        }
    }
    h.stats.rounds_used = rounds_used;
    h.stats.t_augment_s = t_aug.s() - t_vor;

    // ---- final cells + build_all_tables (REF/SPEC.md:397-423) ----
    Timer tt;
    const uint64_t S = h.sites.size();
    std::vector<std::vector<uint32_t>> per(S);
    std::vector<std::vector<Ball>> site_balls(table_fn ? S : 0);  // delegated table job
    std::vector<std::vector<uint32_t>> nbr(S);                    // facet neighbours per cell
    h.cell_box.assign(6 * S, std::nan(""));
    // the device's grid box (p2m_engine.cu: 1.5x the real sites' AABB about its centre, a flat axis
    // padded to 1), grown by a relative 1e-9 so it contains the engine's box despite rounding
    Box gbox;
    {
        Box rb;
        for (uint64_t s = 0; s < S; ++s)
            if (h.kind[s] != P2M_SITE_SENTINEL) rb.add(h.sites[s]);
        for (int c = 0; c < 3; ++c) {
            const double l = comp(rb.lo, c), u = comp(rb.hi, c);
            const double mid = 0.5 * (l + u);
            double hh = 0.75 * (u - l);
            if (!(hh > 0)) hh = 1.0;
            hh *= 1.0 + 1e-9;
            (c == 0 ? gbox.lo.x : c == 1 ? gbox.lo.y : gbox.lo.z) = mid - hh;
            (c == 0 ? gbox.hi.x : c == 1 ? gbox.hi.y : gbox.hi.z) = mid + hh;
        }
    }
    std::vector<uint64_t> ncorner(threads, 0);
    double t_cells = 0.0;
    std::vector<double> tcell(threads, 0.0);
    const double diagD = h.D.diag();
    parallel_for(S, threads, 32, [&](uint64_t b, uint64_t e, int w) {
        CellClipper cc(h.sites, h.tree, outer, h.sentinel_ids, 8, h.eps, kKnn);
        std::vector<V3> corners;
        std::vector<Ball> balls;
        std::vector<uint8_t> mark(NF, 0);
        for (uint64_t s = b; s < e; ++s) {
            if (h.kind[s] == P2M_SITE_SENTINEL) continue;  // empty list (REF/SPEC.md:418)
            Timer tc;
            cc.compute((uint32_t)s, corners, &nbr[s]);
            tcell[w] += tc.s();
            ncorner[w] += corners.size();
            {
                // box of (cell ∩ grid box): the device's exact cell-locate grid only answers points
                // inside the grid box, so clipping first keeps it exact and much tighter for cells
                // that reach the sentinels (outward cones)
                const Box cb = cc.clipped_box((uint32_t)s, gbox);
                double* o = &h.cell_box[6 * s];
                o[0] = cb.lo.x; o[1] = cb.lo.y; o[2] = cb.lo.z; o[3] = cb.hi.x; o[4] = cb.hi.y; o[5] = cb.hi.z;
            }
            const V3 site = h.sites[s];
            balls.clear();
            // closed balls (REF/SPEC.md:95), inflated by a relative 1e-10 and 1e-12*diag(D) so
            // rounding in corners and distances can only add faces (superset, REF/SPEC.md:435)
            auto inflate = [&](double r) { double x = r * (1.0 + 1e-10) + 1e-12 * diagD; return x * x; };
            if (h.kind[s] == P2M_SITE_MESH_VERTEX) {
                // union over corners u of B(u, |u - v|) (Theorem 1, REF/SPEC.md:397-405)
                for (const V3& u : corners) balls.push_back(Ball{u, inflate(std::sqrt(d2(u, site)))});
            } else if (cfg.aux_corner_union) {
                // auxiliary, corner union about the projection: Theorem 1 holds for any centre
                // point, and d(q, M) <= |q - proj| for q in the cell (REF/SPEC.md:413)
                V3 pr = ld3(&h.refs[3 * s]);
                for (const V3& u : corners) balls.push_back(Ball{u, inflate(std::sqrt(d2(u, pr)))});
            } else {
                // auxiliary: B(s, max_u |s-u| + |u-proj|) (REF/SPEC.md:406-414)
                V3 pr = ld3(&h.refs[3 * s]);
                double r = 0.0;
                for (const V3& u : corners) r = std::max(r, std::sqrt(d2(site, u)) + std::sqrt(d2(u, pr)));
                balls.push_back(Ball{site, inflate(r)});
            }
            if (table_fn) { site_balls[s] = balls; continue; }
            h.bvh.balls_query(balls.data(), (int)balls.size(), per[s], mark);
            std::sort(per[s].begin(), per[s].end());
        }
    });
    for (double x : tcell) t_cells += x;
    double t_job = 0.0;
    h.off.assign(S + 1, 0);
    if (table_fn) {
        Timer tj;
        run_table_job(h, site_balls, table_fn, table_ctx);
        t_job = tj.s();
    } else {
        for (uint64_t s = 0; s < S; ++s) h.off[s + 1] = h.off[s] + per[s].size();
        h.lists.resize(h.off[S]);
        for (uint64_t s = 0; s < S; ++s) {
            std::copy(per[s].begin(), per[s].end(), h.lists.begin() + h.off[s]);
            std::vector<uint32_t>().swap(per[s]);
        }
    }
    uint64_t lmax = 0, real = 0;
    for (uint64_t s = 0; s < S; ++s) {
        lmax = std::max<uint64_t>(lmax, h.off[s + 1] - h.off[s]);
        if (h.kind[s] != P2M_SITE_SENTINEL) ++real;
    }
    build_adjacency(h, nbr);
    h.stats.list_entries = h.off[S];
    h.stats.list_max = lmax;
    h.stats.list_avg = real ? (double)h.off[S] / (double)real : 0.0;
    uint64_t nc = 0;
    for (auto x : ncorner) nc += x;
    h.stats.cell_corners = nc;
    h.stats.n_sites = S;
    h.stats.n_aux_sites = S - NV - 8;
    // Table-3 split: "voronoi" = the cell passes of the augmentation rounds plus the final cell
    // construction (thread-summed time rescaled to the final pass's wall time), "tables" = rest
    const double wall = tt.s() - t_job;
    double cell_cpu = t_cells, all_cpu = wall * threads;
    const double cell_wall = all_cpu > 0 ? wall * std::min(1.0, cell_cpu / all_cpu) : 0.0;
    h.stats.t_voronoi_s = t_vor + cell_wall;
    h.stats.t_tables_s = wall - cell_wall + t_job;
    finish_engine(h);
    h.stats.t_total_s = total.s();
    // sentinel guarantee (REF/SPEC.md:250, 287): no sentinel is nearest inside D
    for (int i = 0; i < 10000 + 8; ++i) {
        V3 p;
        if (i < 8) {
            p = V3{(i & 1) ? h.D.hi.x : h.D.lo.x, (i & 2) ? h.D.hi.y : h.D.lo.y, (i & 4) ? h.D.hi.z : h.D.lo.z};
        } else {
            V3 e = h.D.ext();
            p = V3{h.D.lo.x + e.x * u01(99, 0, i), h.D.lo.y + e.y * u01(99, 1, i), h.D.lo.z + e.z * u01(99, 2, i)};
        }
        double dd;
        uint32_t w = h.tree.nearest(p, INFINITY, &dd);
        if (w != UINT32_MAX && h.kind[w] == P2M_SITE_SENTINEL)
            throw GeometryErr("make_bounded_site_set: a sentinel is nearest inside D");
    }
    return hp;
}

}  // namespace p2m
