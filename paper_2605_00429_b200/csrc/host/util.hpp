// util.hpp -- host-side helpers: thread fan-out, counter-based PRNG, error state.
#pragma once

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <string>
#include <thread>
#include <vector>

namespace p2m {

inline int hw_threads(int requested) {
    if (requested > 0) return requested;
    unsigned n = std::thread::hardware_concurrency();
    return n ? (int)n : 1;
}

// Dynamic fan-out over [0, n) in chunks; fn(begin, end, worker).  Per-item work writes to
// disjoint slots (REF/"per-site outputs written to disjoint slots").
inline void parallel_for(uint64_t n, int threads, uint64_t chunk,
                         const std::function<void(uint64_t, uint64_t, int)>& fn) {
    threads = hw_threads(threads);
    if (n == 0) return;
    if (threads == 1 || n <= chunk) { fn(0, n, 0); return; }
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (;;) {
                uint64_t b = next.fetch_add(chunk);
                if (b >= n) break;
                fn(b, std::min(n, b + chunk), t);
            }
        });
    for (auto& th : pool) th.join();
}

// splitmix64 finaliser; the 64-bit splittable seeded PRNG of REF/SPEC.md:650, used in
// counter mode so that every draw is a pure function of (seed, stream, index).
inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t index) {
    return mix64(mix64(seed * 0xD1B54A32D192ED03ull + stream) ^ index);
}
// uniform in [0, 1)
inline double u01(uint64_t seed, uint64_t stream, uint64_t index) {
    return (double)(draw(seed, stream, index) >> 11) * 0x1.0p-53;
}
// standard normal (Box-Muller, host only)
inline double normal01(uint64_t seed, uint64_t stream, uint64_t index) {
    double u1 = 1.0 - u01(seed, stream, 2 * index);  // (0, 1]
    double u2 = u01(seed, stream, 2 * index + 1);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double s() const {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
};

void set_error(const std::string& msg);
std::string get_error();

}  // namespace p2m
