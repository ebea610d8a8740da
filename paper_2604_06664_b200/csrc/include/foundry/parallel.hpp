// Minimal fork-join helper for the host-side tools (pack, save, file staging).
#pragma once

#include <algorithm>
#include <atomic>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

namespace foundry {

inline unsigned default_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? std::min(hw, 32u) : 4u;
}

// Runs fn(i) for i in [0, n) on up to `threads` workers; rethrows the first
// exception after all workers stop.
template <typename Fn>
void parallel_for(size_t n, unsigned threads, Fn&& fn) {
    if (threads == 0) threads = default_threads();
    threads = static_cast<unsigned>(std::min<size_t>(threads, n));
    if (threads <= 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<size_t> next{0};
    std::exception_ptr first;
    std::mutex mu;
    auto body = [&] {
        for (;;) {
            const size_t i = next.fetch_add(1);
            if (i >= n) return;
            try {
                fn(i);
            } catch (...) {
                std::lock_guard lock(mu);
                if (!first) first = std::current_exception();
                next.store(n);
            }
        }
    };
    std::vector<std::thread> pool;
    pool.reserve(threads - 1);
    for (unsigned t = 1; t < threads; ++t) pool.emplace_back(body);
    body();
    for (auto& t : pool) t.join();
    if (first) std::rethrow_exception(first);
}

}  // namespace foundry
