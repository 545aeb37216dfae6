// query_demo.cpp -- the C++ build-then-query API end to end (reference-style host code).
//   make examples/query_demo && ./examples/query_demo [config 1..5] [n_queries]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../include/p2m_engine.hpp"

int main(int argc, char** argv) {
    const int cfg = argc > 1 ? std::atoi(argv[1]) : 1;
    const uint64_t n = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 100000;
    double* v = nullptr;
    uint32_t* f = nullptr;
    uint64_t nv = 0, nf = 0;
    p2m::check(p2m_mesh_config(cfg, &v, &nv, &f, &nf));
    std::vector<p2m::Vec3> V(reinterpret_cast<p2m::Vec3*>(v), reinterpret_cast<p2m::Vec3*>(v) + nv);
    std::vector<uint32_t> F(f, f + 3 * nf);
    p2m_free(v);
    p2m_free(f);
    std::vector<p2m::Vec3> q(n);
    p2m::check(p2m_gen_queries(cfg, reinterpret_cast<const double*>(V.data()), nv, F.data(), nf, 0, n,
                               reinterpret_cast<double*>(q.data())));
    auto t0 = std::chrono::steady_clock::now();
    p2m::HostEngine host = p2m::HostEngine::build(V, F);
    auto t1 = std::chrono::steady_clock::now();
    p2m::Engine eng(host);
    eng.batch_query(q);  // warm-up
    auto t2 = std::chrono::steady_clock::now();
    p2m::BatchResult r = eng.batch_query(q);
    auto t3 = std::chrono::steady_clock::now();
    const p2m_build_stats st = host.stats();
    std::printf("config %d: %llu faces, %llu sites, build %.2f s, %llu queries in %.3f ms (host buffers)\n", cfg,
                (unsigned long long)st.n_faces, (unsigned long long)st.n_sites,
                std::chrono::duration<double>(t1 - t0).count(), (unsigned long long)n,
                std::chrono::duration<double, std::milli>(t3 - t2).count());
    std::printf("q[0] = (%.6f %.6f %.6f): distance %.17g face %u site %u flags %u\n", q[0].x, q[0].y, q[0].z,
                r.distance[0], r.face[0], r.site[0], r.flags[0]);
    std::printf("candidates/query %.1f, exact/query %.1f\n", (double)r.counters.candidates_visited / n,
                (double)r.counters.exact_evaluations / n);
    return 0;
}
