// Host-side data parallelism shared by the plugin adapter and the wire
// codec: plain std::thread fan-out over index ranges.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <thread>
#include <vector>

namespace sfxb {
namespace hostpar {

// SFXB_HOST_THREADS, else the hardware threads (at most 32)
inline unsigned host_threads() {
    static unsigned n = [] {
        if (const char *e = std::getenv("SFXB_HOST_THREADS")) return (unsigned)std::max(1, std::atoi(e));
        unsigned h = std::thread::hardware_concurrency();
        return h ? std::min(h, 32u) : 4u;
    }();
    return n;
}

// f(lo, hi) over [0, n) on host_threads() threads; ranges below `grain`
// items run inline
template <typename F>
void parallel_for(size_t n, F &&f, size_t grain = 4096) {
    const unsigned T = host_threads();
    if (n < grain || n < 2 || T <= 1) {
        f(size_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    const size_t chunk = (n + T - 1) / T;
    for (unsigned t = 0; t < T; ++t) {
        size_t lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&, lo, hi] { f(lo, hi); });
    }
    for (auto &th : pool) th.join();
}

} // namespace hostpar
} // namespace sfxb
