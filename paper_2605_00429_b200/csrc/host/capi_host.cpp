// capi_host.cpp -- C ABI of libp2m_host.so (declared in include/p2m.h): builder, EngineIndexFile,
// synthetic workload generators, and the shared thread-local error string.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

#include "../../../include/p2m.h"
#include "builder.hpp"
#include "meshgen.hpp"
#include "util.hpp"

#define P2M_API extern "C" __attribute__((visibility("default")))

namespace p2m {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
std::string get_error() { return g_err; }
}  // namespace p2m

struct p2m_host_engine {
    std::unique_ptr<p2m::HostEngine> h;
};

using p2m::set_error;

template <class F>
static int guarded(F&& fn) {
    try {
        p2m::g_err.clear();
        return fn();
    } catch (const p2m::GeometryErr& e) {
        set_error(e.what());
        return P2M_ERR_GEOMETRY;
    } catch (const std::invalid_argument& e) {
        set_error(e.what());
        return P2M_ERR_INVALID;
    } catch (const std::bad_alloc&) {
        set_error("out of host memory");
        return P2M_ERR_OOM;
    } catch (const std::exception& e) {
        set_error(e.what());
        return P2M_ERR_INTERNAL;
    }
}

P2M_API const char* p2m_last_error(void) { return p2m::g_err.c_str(); }

// internal hook for libp2m_cuda.so (same thread-local string)
P2M_API void p2m_set_last_error_internal(const char* msg) { set_error(msg ? msg : ""); }

P2M_API void p2m_build_config_default(p2m_build_config* c) {
    if (!c) return;
    c->augment = 1;
    c->alpha = 4.0;
    c->k = 24;
    c->rho = 0.75;
    c->max_rounds = 3;
    c->domain_scale = 10.0;
    c->n_threads = 0;
    c->strict_mesh = 0;
    c->aux_corner_union = 1;
}

P2M_API int p2m_build(const double* vertices, uint64_t n_vertices, const uint32_t* faces,
                      uint64_t n_faces, const p2m_build_config* cfg, p2m_host_engine** out) {
    return guarded([&] {
        if (!vertices || !faces || !out) throw std::invalid_argument("p2m_build: null pointer");
        p2m_build_config c;
        if (cfg) c = *cfg; else p2m_build_config_default(&c);
        auto h = p2m::build_engine(vertices, n_vertices, faces, n_faces, c);
        *out = new p2m_host_engine{std::move(h)};
        return (int)P2M_OK;
    });
}

P2M_API int p2m_build_with(const double* vertices, uint64_t n_vertices, const uint32_t* faces,
                           uint64_t n_faces, const p2m_build_config* cfg, p2m_table_fn fn, void* ctx,
                           p2m_host_engine** out) {
    return guarded([&] {
        if (!vertices || !faces || !out) throw std::invalid_argument("p2m_build_with: null pointer");
        p2m_build_config c;
        if (cfg) c = *cfg; else p2m_build_config_default(&c);
        auto h = p2m::build_engine(vertices, n_vertices, faces, n_faces, c, fn, ctx);
        *out = new p2m_host_engine{std::move(h)};
        return (int)P2M_OK;
    });
}

P2M_API void p2m_host_engine_destroy(p2m_host_engine* h) { delete h; }

P2M_API int p2m_host_engine_desc(const p2m_host_engine* he, p2m_engine_desc* d) {
    return guarded([&] {
        if (!he || !d) throw std::invalid_argument("p2m_host_engine_desc: null pointer");
        const p2m::HostEngine& h = *he->h;
        d->n_sites = h.sites.size();
        d->site_xyz = h.site_xyz.data();
        d->site_kind = h.kind.data();
        d->n_faces = h.F.size() / 3;
        d->tri_xyz = h.tri.data();
        d->face_sphere = h.sphere.data();
        d->list_offsets = h.off.data();
        d->list_faces = h.lists.data();
        d->site_cell_box = h.cell_box.empty() ? nullptr : h.cell_box.data();
        d->site_ref_xyz = h.refs.empty() ? nullptr : h.refs.data();
        d->adj_offsets = h.adj_off.empty() ? nullptr : h.adj_off.data();
        d->adj_sites = h.adj_off.empty() ? nullptr : h.adj.data();
        d->domain_min[0] = h.D.lo.x; d->domain_min[1] = h.D.lo.y; d->domain_min[2] = h.D.lo.z;
        d->domain_max[0] = h.D.hi.x; d->domain_max[1] = h.D.hi.y; d->domain_max[2] = h.D.hi.z;
        return (int)P2M_OK;
    });
}

P2M_API int p2m_host_engine_stats(const p2m_host_engine* he, p2m_build_stats* s) {
    if (!he || !s) { set_error("p2m_host_engine_stats: null pointer"); return P2M_ERR_INVALID; }
    *s = he->h->stats;
    return P2M_OK;
}

P2M_API int p2m_host_engine_mesh(const p2m_host_engine* he, const double** v, uint64_t* nv,
                                 const uint32_t** f, uint64_t* nf) {
    if (!he) { set_error("p2m_host_engine_mesh: null engine"); return P2M_ERR_INVALID; }
    if (v) *v = he->h->V.data();
    if (nv) *nv = he->h->V.size() / 3;
    if (f) *f = he->h->F.data();
    if (nf) *nf = he->h->F.size() / 3;
    return P2M_OK;
}

P2M_API int p2m_host_engine_site_refs(const p2m_host_engine* he, const double** refs) {
    if (!he || !refs) { set_error("p2m_host_engine_site_refs: null pointer"); return P2M_ERR_INVALID; }
    *refs = he->h->refs.data();
    return P2M_OK;
}

P2M_API int p2m_host_engine_cell_corners(const p2m_host_engine* he, uint64_t site, double* out,
                                         uint64_t capacity, uint64_t* n) {
    return guarded([&] {
        if (!he || !n) throw std::invalid_argument("p2m_host_engine_cell_corners: null pointer");
        const p2m::HostEngine& h = *he->h;
        if (site >= h.sites.size()) throw std::invalid_argument("cell_corners: site out of range");
        if (h.kind[site] == P2M_SITE_SENTINEL) throw std::invalid_argument("cell_corners: sentinel site");
        std::vector<p2m::V3> c;
        p2m::cell_corners(h, (uint32_t)site, c);
        *n = c.size();
        for (uint64_t i = 0; i < c.size() && i < capacity && out; ++i) {
            out[3 * i] = c[i].x; out[3 * i + 1] = c[i].y; out[3 * i + 2] = c[i].z;
        }
        return (int)P2M_OK;
    });
}

P2M_API int p2m_host_closest_point(const p2m_host_engine* he, const double* q, double* d2, double* p,
                                   uint32_t* face) {
    if (!he || !q) { set_error("p2m_host_closest_point: null pointer"); return P2M_ERR_INVALID; }
    double dd;
    p2m::V3 pp;
    uint32_t f = he->h->bvh.closest(p2m::ld3(q), &dd, &pp);
    if (d2) *d2 = dd;
    if (p) { p[0] = pp.x; p[1] = pp.y; p[2] = pp.z; }
    if (face) *face = f;
    return P2M_OK;
}

// ---------------------------------------------------------------------------------------------
// EngineIndexFile (REF/SPEC.md:588-591): magic "P2MX", LE u32 version, mesh hash, D, sites
// (kind, position, reference), per-site table offsets + face ids, config echo.  The BVH and the
// NNS index are rebuilt on load (REF/SPEC.md:639).
static const uint32_t kFileVersion = 4;  // v2 cell boxes, v3 Delaunay adjacency, v4 field-by-field config/stats

// config and stats field by field with explicit widths (little-endian), never as struct dumps
template <class IO>
static void cfg_fields(p2m_build_config& c, IO&& io) {
    io(c.augment); io(c.alpha); io(c.k); io(c.rho); io(c.max_rounds); io(c.domain_scale); io(c.n_threads);
    io(c.strict_mesh); io(c.aux_corner_union);
}
template <class IO>
static void stats_fields(p2m_build_stats& t, IO&& io) {
    io(t.n_input_vertices); io(t.n_input_faces); io(t.n_vertices); io(t.n_faces); io(t.merged_vertices);
    io(t.removed_faces); io(t.n_sites); io(t.n_aux_sites); io(t.rounds_used); io(t.mean_edge); io(t.tau);
    io(t.list_entries); io(t.list_max); io(t.list_avg); io(t.t_voronoi_s); io(t.t_augment_s); io(t.t_tables_s);
    io(t.t_total_s); io(t.cell_corners);
}

P2M_API int p2m_host_engine_save(const p2m_host_engine* he, const char* path) {
    return guarded([&] {
        if (!he || !path) throw std::invalid_argument("p2m_host_engine_save: null pointer");
        const p2m::HostEngine& h = *he->h;
        FILE* fp = std::fopen(path, "wb");
        if (!fp) { set_error(std::string("cannot open ") + path); return (int)P2M_ERR_IO; }
        bool ok = true;
        auto w = [&](const void* p, size_t n) { ok = ok && std::fwrite(p, 1, n, fp) == n; };
        w("P2MX", 4);
        w(&kFileVersion, 4);
        w(&h.mesh_hash, 8);
        double dom[6] = {h.D.lo.x, h.D.lo.y, h.D.lo.z, h.D.hi.x, h.D.hi.y, h.D.hi.z};
        w(dom, sizeof dom);
        p2m_build_config cfg = h.cfg;
        p2m_build_stats st = h.stats;
        cfg_fields(cfg, [&](auto& x) { w(&x, sizeof x); });
        stats_fields(st, [&](auto& x) { w(&x, sizeof x); });
        uint64_t S = h.sites.size();
        w(&S, 8);
        w(h.kind.data(), S);
        w(h.site_xyz.data(), 24 * S);
        w(h.refs.data(), 24 * S);
        w(h.sentinel_ids, sizeof h.sentinel_ids);
        w(h.off.data(), 8 * (S + 1));
        w(h.lists.data(), 4 * h.lists.size());
        w(h.cell_box.data(), 8 * h.cell_box.size());
        const uint64_t na = h.adj.size();
        w(&na, 8);
        w(h.adj_off.data(), 8 * h.adj_off.size());
        w(h.adj.data(), 4 * na);
        w("XM2P", 4);
        ok = (std::fclose(fp) == 0) && ok;
        if (!ok) { set_error("write failed"); return (int)P2M_ERR_IO; }
        return (int)P2M_OK;
    });
}

P2M_API int p2m_host_engine_load(const char* path, const double* vertices, uint64_t n_vertices,
                                 const uint32_t* faces, uint64_t n_faces, p2m_host_engine** out) {
    return guarded([&] {
        if (!path || !vertices || !faces || !out) throw std::invalid_argument("p2m_host_engine_load: null pointer");
        FILE* fp = std::fopen(path, "rb");
        if (!fp) { set_error(std::string("cannot open ") + path); return (int)P2M_ERR_IO; }
        bool ok = true;
        auto r = [&](void* p, size_t n) { ok = ok && std::fread(p, 1, n, fp) == n; };
        char magic[4] = {0};
        uint32_t ver = 0;
        r(magic, 4);
        r(&ver, 4);
        if (!ok || std::memcmp(magic, "P2MX", 4) != 0) { std::fclose(fp); set_error("not an EngineIndexFile (magic)"); return (int)P2M_ERR_IO; }
        if (ver != kFileVersion) { std::fclose(fp); set_error("EngineIndexFile version mismatch"); return (int)P2M_ERR_IO; }
        auto hp = std::make_unique<p2m::HostEngine>();
        p2m::HostEngine& h = *hp;
        uint64_t hash = 0;
        r(&hash, 8);
        double dom[6];
        r(dom, sizeof dom);
        h.cfg = p2m_build_config{};
        h.stats = p2m_build_stats{};
        cfg_fields(h.cfg, [&](auto& x) { r(&x, sizeof x); });
        stats_fields(h.stats, [&](auto& x) { r(&x, sizeof x); });
        if (!ok) { std::fclose(fp); set_error("EngineIndexFile truncated (header)"); return (int)P2M_ERR_IO; }
        if (!(h.cfg.alpha > 0) || h.cfg.k < 1 || !(h.cfg.rho > 0) || h.cfg.max_rounds < 1 || !(h.cfg.domain_scale >= 1)) {
            std::fclose(fp); set_error("EngineIndexFile corrupt (config)"); return (int)P2M_ERR_IO;
        }
        // re-validate the caller's mesh exactly as the build did and compare the hash
        p2m_build_config c = h.cfg;
        auto probe = p2m::build_engine_mesh_only(vertices, n_vertices, faces, n_faces, c);
        if (probe->mesh_hash != hash) { std::fclose(fp); set_error("EngineIndexFile mesh hash mismatch"); return (int)P2M_ERR_IO; }
        h.V = std::move(probe->V);
        h.F = std::move(probe->F);
        h.tri = std::move(probe->tri);
        h.sphere = std::move(probe->sphere);
        h.aabb = probe->aabb;
        h.mesh_hash = hash;
        h.D.lo = p2m::V3{dom[0], dom[1], dom[2]};
        h.D.hi = p2m::V3{dom[3], dom[4], dom[5]};
        h.sentinel_box = h.D.scaled(4.0, 0.0);
        h.eps = 1e-12 * h.D.diag();
        uint64_t S = 0;
        r(&S, 8);
        if (!ok || S > (1ull << 32)) { std::fclose(fp); set_error("EngineIndexFile truncated (sites)"); return (int)P2M_ERR_IO; }
        h.kind.resize(S);
        h.site_xyz.resize(3 * S);
        h.refs.resize(3 * S);
        h.off.resize(S + 1);
        r(h.kind.data(), S);
        r(h.site_xyz.data(), 24 * S);
        r(h.refs.data(), 24 * S);
        r(h.sentinel_ids, sizeof h.sentinel_ids);
        r(h.off.data(), 8 * (S + 1));
        if (!ok || h.off[S] > (1ull << 36)) { std::fclose(fp); set_error("EngineIndexFile truncated (tables)"); return (int)P2M_ERR_IO; }
        h.lists.resize(h.off[S]);
        r(h.lists.data(), 4 * h.lists.size());
        h.cell_box.resize(6 * S);
        r(h.cell_box.data(), 8 * h.cell_box.size());
        uint64_t na = 0;
        r(&na, 8);
        if (!ok || na > (1ull << 36)) { std::fclose(fp); set_error("EngineIndexFile truncated (adjacency)"); return (int)P2M_ERR_IO; }
        h.adj_off.resize(S + 1);
        h.adj.resize(na);
        r(h.adj_off.data(), 8 * (S + 1));
        r(h.adj.data(), 4 * na);
        if (ok && (h.adj_off[0] != 0 || h.adj_off[S] != na)) { std::fclose(fp); set_error("EngineIndexFile corrupt (adjacency)"); return (int)P2M_ERR_IO; }
        char tail[4] = {0};
        r(tail, 4);
        std::fclose(fp);
        if (!ok || std::memcmp(tail, "XM2P", 4) != 0) { set_error("EngineIndexFile truncated"); return (int)P2M_ERR_IO; }
        // contents: every id and offset within range before anything uses them (a corrupt or foreign
        // file must fail here, not read out of bounds in the table or query paths)
        const uint64_t NF = h.F.size() / 3;
        auto corrupt = [&](const char* what) { set_error(std::string("EngineIndexFile corrupt (") + what + ")"); return (int)P2M_ERR_IO; };
        if (h.off[0] != 0) return corrupt("table offsets");
        for (uint64_t i = 0; i < S; ++i) if (h.off[i] > h.off[i + 1]) return corrupt("table offsets");
        for (uint32_t f : h.lists) if (f >= NF) return corrupt("face ids");
        for (uint64_t i = 0; i < S; ++i) if (h.adj_off[i] > h.adj_off[i + 1]) return corrupt("adjacency offsets");
        for (uint32_t a : h.adj) if (a >= S) return corrupt("adjacency ids");
        uint64_t n_sent = 0;
        for (uint64_t i = 0; i < S; ++i) {
            if (h.kind[i] > 2) return corrupt("site kinds");
            if (!std::isfinite(h.site_xyz[3 * i]) || !std::isfinite(h.site_xyz[3 * i + 1]) || !std::isfinite(h.site_xyz[3 * i + 2]))
                return corrupt("site positions");
            n_sent += h.kind[i] == 1;
        }
        for (uint32_t id : h.sentinel_ids) if (id >= S || h.kind[id] != 1) return corrupt("sentinel ids");
        if (n_sent != sizeof h.sentinel_ids / sizeof h.sentinel_ids[0]) return corrupt("sentinel count");
        h.sites.resize(S);
        for (uint64_t i = 0; i < S; ++i) h.sites[i] = p2m::ld3(&h.site_xyz[3 * i]);
        h.bvh.build(h.tri.data(), h.F.size() / 3, 4);
        p2m::finish_engine(h);
        *out = new p2m_host_engine{std::move(hp)};
        return (int)P2M_OK;
    });
}

P2M_API int p2m_delaunay_adjacency(const double* xyz, uint64_t n, uint64_t** off, uint32_t** adj) {
    return guarded([&] {
        if (!xyz || !off || !adj || n == 0) throw std::invalid_argument("p2m_delaunay_adjacency: bad argument");
        std::vector<uint64_t> o;
        std::vector<uint32_t> a;
        p2m::delaunay_adjacency(xyz, n, 0, o, a);
        *off = (uint64_t*)std::malloc(8 * o.size());
        *adj = (uint32_t*)std::malloc(4 * std::max<size_t>(1, a.size()));
        if (!*off || !*adj) { std::free(*off); std::free(*adj); *off = nullptr; *adj = nullptr; throw std::bad_alloc(); }
        std::memcpy(*off, o.data(), 8 * o.size());
        if (!a.empty()) std::memcpy(*adj, a.data(), 4 * a.size());
        return (int)P2M_OK;
    });
}

// ---------------------------------------------------------------------------------------------
static int export_mesh(const p2m::Mesh& m, double** v, uint64_t* nv, uint32_t** f, uint64_t* nf) {
    *v = (double*)std::malloc(sizeof(double) * m.v.size());
    *f = (uint32_t*)std::malloc(sizeof(uint32_t) * m.f.size());
    if (!*v || !*f) { std::free(*v); std::free(*f); set_error("out of host memory"); return P2M_ERR_OOM; }
    std::memcpy(*v, m.v.data(), sizeof(double) * m.v.size());
    std::memcpy(*f, m.f.data(), sizeof(uint32_t) * m.f.size());
    *nv = m.v.size() / 3;
    *nf = m.f.size() / 3;
    return P2M_OK;
}

P2M_API int p2m_mesh_config(int cfg, double** v, uint64_t* nv, uint32_t** f, uint64_t* nf) {
    return guarded([&] {
        if (!v || !nv || !f || !nf) throw std::invalid_argument("p2m_mesh_config: null pointer");
        return export_mesh(p2m::mesh_config(cfg), v, nv, f, nf);
    });
}

P2M_API int p2m_mesh_icosphere(int level, double** v, uint64_t* nv, uint32_t** f, uint64_t* nf) {
    return guarded([&] {
        if (!v || !nv || !f || !nf || level < 0 || level > 10) throw std::invalid_argument("p2m_mesh_icosphere: bad argument");
        return export_mesh(p2m::icosphere(level), v, nv, f, nf);
    });
}

P2M_API int p2m_gen_queries(int cfg, const double* v, uint64_t nv, const uint32_t* f, uint64_t nf,
                            uint64_t first, uint64_t count, double* out) {
    return guarded([&] {
        if (!v || !f || (!out && count)) throw std::invalid_argument("p2m_gen_queries: null pointer");
        p2m::gen_queries(cfg, v, nv, f, nf, first, count, out);
        return (int)P2M_OK;
    });
}

P2M_API int p2m_gen_uniform(uint64_t seed, const double* lo, const double* hi, uint64_t first,
                            uint64_t count, double* out) {
    return guarded([&] {
        if (!lo || !hi || (!out && count)) throw std::invalid_argument("p2m_gen_uniform: null pointer");
        p2m::gen_uniform(seed, lo, hi, first, count, out);
        return (int)P2M_OK;
    });
}

P2M_API void p2m_free(void* p) { std::free(p); }
