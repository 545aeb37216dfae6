// p2m_engine.hpp -- C++ build-then-query API over the C ABI (include/p2m.h).
//
// Mirrors the reference's engine ops (REF = /root/reference, spec-only beyond geometry):
//   p2m::HostEngine::build   <- cmd_build pipeline           REF/SPEC.md:598-606
//   p2m::Engine(host, gpus)  <- build_nns_index + hand-off    REF/SPEC.md:473-481
//   Engine::nearest_site     <- nearest_site                  REF/SPEC.md:482-487
//   Engine::query_distance   <- query_distance                REF/SPEC.md:488-496
//   Engine::batch_query      <- batch_query                   REF/SPEC.md:497-505
// Errors surface as p2m::Error (a std::runtime_error carrying the P2M_ERR_* code), the analogue of
// p2mx::GeometryError (REF/proj/include/p2mx/geom.hpp:88-91); out-of-domain rows are never errors
// (REF/SPEC.md:611), they are answered exactly and flagged.
// Link: -Lpaper_2605_00429_b200/lib -lp2m_cuda -lp2m_host
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "p2m.h"

namespace p2m {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void check(int rc) {
    if (rc != P2M_OK) throw Error(rc, std::string("p2m: ") + p2m_last_error());
}

struct Vec3 {
    double x, y, z;
};

struct QueryResult {  // REF/SPEC.md:467-470
    double distance;
    Vec3 closest;
    uint32_t face;
    uint32_t site;
    uint32_t flags;
    bool fallback() const { return (flags & P2M_FLAG_FALLBACK) != 0; }
};

struct BatchResult {
    std::vector<double> distance;
    std::vector<Vec3> closest;
    std::vector<uint32_t> face, site, flags;
    p2m_counters counters{};
};

class HostEngine {
   public:
    static HostEngine build(const std::vector<Vec3>& vertices, const std::vector<uint32_t>& faces,
                            const p2m_build_config* cfg = nullptr) {
        HostEngine e;
        check(p2m_build(reinterpret_cast<const double*>(vertices.data()), vertices.size(), faces.data(),
                        faces.size() / 3, cfg, &e.h_));
        return e;
    }
    static HostEngine load(const std::string& path, const std::vector<Vec3>& vertices,
                           const std::vector<uint32_t>& faces) {
        HostEngine e;
        check(p2m_host_engine_load(path.c_str(), reinterpret_cast<const double*>(vertices.data()),
                                   vertices.size(), faces.data(), faces.size() / 3, &e.h_));
        return e;
    }
    void save(const std::string& path) const { check(p2m_host_engine_save(h_, path.c_str())); }
    p2m_build_stats stats() const {
        p2m_build_stats s;
        check(p2m_host_engine_stats(h_, &s));
        return s;
    }
    p2m_engine_desc desc() const {
        p2m_engine_desc d;
        check(p2m_host_engine_desc(h_, &d));
        return d;
    }
    HostEngine(HostEngine&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    HostEngine& operator=(HostEngine&& o) noexcept {
        std::swap(h_, o.h_);
        return *this;
    }
    HostEngine(const HostEngine&) = delete;
    HostEngine& operator=(const HostEngine&) = delete;
    ~HostEngine() { p2m_host_engine_destroy(h_); }

   private:
    HostEngine() = default;
    p2m_host_engine* h_ = nullptr;
};

class Engine {
   public:
    explicit Engine(const HostEngine& host, const std::vector<int>& devices = {0}) {
        p2m_engine_desc d = host.desc();
        check(p2m_engine_create(&d, (int)devices.size(), devices.data(), &e_));
    }
    // straight from a device image (p2m_engine_load): no host engine, no re-packing
    static Engine load(const std::string& path, const std::vector<int>& devices = {0}) {
        Engine e;
        check(p2m_engine_load(path.c_str(), (int)devices.size(), devices.data(), &e.e_));
        return e;
    }
    void save(const std::string& path) const { check(p2m_engine_save(e_, path.c_str())); }
    Engine(Engine&& o) noexcept : e_(o.e_) { o.e_ = nullptr; }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ~Engine() { p2m_engine_destroy(e_); }

    BatchResult batch_query(const std::vector<Vec3>& q) const {
        BatchResult r;
        const size_t n = q.size();
        r.distance.resize(n); r.closest.resize(n); r.face.resize(n); r.site.resize(n); r.flags.resize(n);
        check(p2m_query(e_, reinterpret_cast<const double*>(q.data()), n, r.distance.data(),
                        reinterpret_cast<double*>(r.closest.data()), r.face.data(), r.site.data(),
                        r.flags.data(), &r.counters));
        return r;
    }
    QueryResult query_distance(const Vec3& q) const {
        BatchResult b = batch_query({q});
        return QueryResult{b.distance[0], b.closest[0], b.face[0], b.site[0], b.flags[0]};
    }
    uint32_t nearest_site(const Vec3& q) const { return query_distance(q).site; }
    p2m_engine* handle() const { return e_; }

   private:
    Engine() = default;
    p2m_engine* e_ = nullptr;
};

}  // namespace p2m
