// Host-side data parallelism shared by the plugin adapter and the wire
// codec: plain std::thread fan-out over index ranges.
#pragma once
#include <malloc.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
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

// While alive, glibc grows each thread's malloc heap in 128 MB steps instead
// of 128 KB.  Writing millions of fresh mpz limb arrays (≈1 GB per tree) on
// all host threads otherwise serialises on the heap-growth mprotect calls
// (parse of 2M ciphertexts: import 0.69 -> 0.28 s on 8 threads).  Left alone
// when the user tuned M_TOP_PAD (MALLOC_TOP_PAD_ or GLIBC_TUNABLES) or sets
// SFXB_HOST_TOP_PAD=0.
//
// Scopes nest and overlap across threads (parties call their plugins
// concurrently in the reference's threaded mode, federation.cpp:509-516): a
// process-wide count under a mutex raises the step on the first entry and
// restores glibc's default (128 KiB) on the last exit only, so one party's
// exit never shrinks the step under another party still writing.  Side
// effect (glibc): any mallopt(M_TOP_PAD) call also disables the dynamic mmap
// threshold for the rest of the process; an application
// that cannot accept that sets SFXB_HOST_TOP_PAD=0.
class TopPadScope {
  public:
    explicit TopPadScope(size_t bytes_to_allocate) {
        static const bool allowed = [] {
            if (std::getenv("MALLOC_TOP_PAD_")) return false;
            if (const char *t = std::getenv("GLIBC_TUNABLES"); t && std::strstr(t, "top_pad")) return false;
            const char *e = std::getenv("SFXB_HOST_TOP_PAD");
            return !(e && std::atoi(e) == 0);
        }();
        on_ = allowed && bytes_to_allocate >= (size_t(16) << 20);
        if (!on_) return;
        std::lock_guard<std::mutex> lk(state().mu);
        if (state().depth++ == 0) mallopt(M_TOP_PAD, 128 << 20);
    }
    ~TopPadScope() {
        if (!on_) return;
        std::lock_guard<std::mutex> lk(state().mu);
        if (--state().depth == 0) mallopt(M_TOP_PAD, 128 * 1024);
    }
    TopPadScope(const TopPadScope &) = delete;
    TopPadScope &operator=(const TopPadScope &) = delete;

  private:
    struct Shared {
        std::mutex mu;
        int depth = 0;
    };
    static Shared &state() {
        static Shared s;
        return s;
    }
    bool on_ = false;
};

} // namespace hostpar
} // namespace sfxb
