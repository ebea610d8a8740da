// Checks foundry::parallel_for's worker pool: results, exceptions, nested and
// concurrent calls, and a forked child. Built and run by tests/test_parallel_pool.py.
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <numeric>
#include <stdexcept>

#include "foundry/parallel.hpp"

using foundry::parallel_for;

static int fail(const char* what) {
    std::printf("FAIL %s\n", what);
    return 1;
}

static bool sum_ok(size_t n, unsigned threads) {
    std::vector<uint64_t> v(n, 0);
    parallel_for(n, threads, [&](size_t i) { v[i] = i * 3 + 1; });
    uint64_t s = std::accumulate(v.begin(), v.end(), uint64_t(0));
    return s == 3 * (uint64_t(n) * (n - 1) / 2) + n;
}

int main() {
    for (int r = 0; r < 200; ++r)
        if (!sum_ok(1000 + r, 0)) return fail("sum");
    if (!sum_ok(100000, 3)) return fail("sum, 3 threads");
    if (!sum_ok(64, 64)) return fail("sum, oversubscribed");
    try {  // the first exception surfaces after every worker stopped
        parallel_for(10000, 0, [&](size_t i) {
            if (i == 777) throw std::runtime_error("boom");
        });
        return fail("no exception");
    } catch (const std::runtime_error& e) {
        if (std::string(e.what()) != "boom") return fail("wrong exception");
    }
    if (!sum_ok(5000, 0)) return fail("pool after an exception");
    std::atomic<uint64_t> nested{0};  // inner calls find the pool busy
    parallel_for(16, 0, [&](size_t) { parallel_for(100, 4, [&](size_t j) { nested += j; }); });
    if (nested != 16 * 4950) return fail("nested");
    std::atomic<int> bad{0};  // concurrent callers on their own threads
    std::vector<std::thread> ts;
    for (int t = 0; t < 4; ++t)
        ts.emplace_back([&] {
            for (int r = 0; r < 50; ++r)
                if (!sum_ok(2000 + r, 0)) ++bad;
        });
    for (auto& t : ts) t.join();
    if (bad) return fail("concurrent");
    const pid_t pid = fork();  // the child has no workers: the caller drains alone
    if (pid == 0) _exit(sum_ok(10000, 0) && sum_ok(20000, 0) ? 0 : 3);
    int status = 0;
    waitpid(pid, &status, 0);
    if (!WIFEXITED(status) || WEXITSTATUS(status) != 0) return fail("forked child");
    if (!sum_ok(30000, 0)) return fail("parent after fork");
    std::printf("ok\n");
    return 0;
}
