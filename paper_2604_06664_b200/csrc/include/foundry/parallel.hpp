// Fork-join helper for the host-side work (pack, save, staging, restore).
//
// parallel_for runs on a persistent worker pool: spawning and joining 15 threads
// per call cost 0.3-1 ms, which the GPU packer paid three times per archive. One
// job runs on the pool at a time; a call made while the pool is busy (another
// thread's job, or a nested call) spawns its own threads as before. The caller
// always drains the job itself and waits only for the workers that joined it,
// so a pool without workers (a forked child) degrades to a serial loop.
#pragma once

#include <pthread.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <new>
#include <thread>
#include <type_traits>
#include <vector>

namespace foundry {

inline unsigned default_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? std::min(hw, 32u) : 4u;
}

namespace detail {

struct ForJob {
    void (*call)(void*, size_t) = nullptr;
    void* ctx = nullptr;
    size_t n = 0;
    unsigned max_helpers = 0;
    std::atomic<size_t> next{0};
    std::mutex mu;
    std::exception_ptr first;

    void drain() {
        for (;;) {
            const size_t i = next.fetch_add(1);
            if (i >= n) return;
            try {
                call(ctx, i);
            } catch (...) {
                std::lock_guard lock(mu);
                if (!first) first = std::current_exception();
                next.store(n);
            }
        }
    }
};

class WorkerPool {
public:
    static WorkerPool& get() {
        static WorkerPool* p = [] {  // never destroyed: its threads are detached
            auto* w = new WorkerPool;
            pthread_atfork([] { get().mu_.lock(); }, [] { get().mu_.unlock(); }, [] { get().after_fork_child(); });
            return w;
        }();
        return *p;
    }

    // Runs the job on the calling thread plus up to job.max_helpers workers;
    // false (nothing run) when another job holds the pool.
    bool run(ForJob& job) {
        if (busy_.exchange(true, std::memory_order_acquire)) return false;
        {
            std::lock_guard lk(mu_);
            start_workers_locked();
            job_ = &job;
            joined_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        job.drain();
        {
            std::unique_lock lk(mu_);
            job_ = nullptr;  // closed: no worker joins from here on
            done_.wait(lk, [&] { return in_flight_ == 0; });
        }
        busy_.store(false, std::memory_order_release);
        return true;
    }

private:
    void start_workers_locked() {
        if (started_) return;
        started_ = true;
        const unsigned n = default_threads() > 1 ? default_threads() - 1 : 0;
        for (unsigned i = 0; i < n; ++i) {
            try {
                std::thread([this, g = gen_] { loop(g); }).detach();
            } catch (...) {
                break;  // fewer workers: the caller drains the rest
            }
        }
    }

    void loop(uint64_t seen) {  // seen: the generation before the first job
        std::unique_lock lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            ForJob* j = job_;
            if (!j || joined_ >= j->max_helpers) continue;
            ++joined_;
            ++in_flight_;
            lk.unlock();
            j->drain();
            lk.lock();
            if (--in_flight_ == 0) done_.notify_all();
        }
    }

    // the child has no workers and may have inherited a half-run job's state
    void after_fork_child() {
        new (&mu_) std::mutex;
        new (&cv_) std::condition_variable;
        new (&done_) std::condition_variable;
        job_ = nullptr;
        joined_ = in_flight_ = 0;
        started_ = false;
        busy_.store(false);
    }

    std::mutex mu_;
    std::condition_variable cv_, done_;
    std::atomic<bool> busy_{false};
    ForJob* job_ = nullptr;
    uint64_t gen_ = 0;
    unsigned joined_ = 0, in_flight_ = 0;
    bool started_ = false;
};

}  // namespace detail

// Runs fn(i) for i in [0, n) on up to `threads` workers (the caller included);
// rethrows the first exception after all workers stop.
template <typename Fn>
void parallel_for(size_t n, unsigned threads, Fn&& fn) {
    if (threads == 0) threads = default_threads();
    threads = static_cast<unsigned>(std::min<size_t>(threads, n));
    static const bool no_pool = std::getenv("FOUNDRY_NO_THREAD_POOL") != nullptr;  // diagnostics
    const bool oversubscribed = no_pool || threads > default_threads();  // e.g. threads blocked in the driver
    if (threads <= 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    detail::ForJob job;
    job.call = [](void* ctx, size_t i) { (*static_cast<std::remove_reference_t<Fn>*>(ctx))(i); };
    job.ctx = const_cast<void*>(static_cast<const void*>(&fn));
    job.n = n;
    job.max_helpers = threads - 1;
    if (oversubscribed || !detail::WorkerPool::get().run(job)) {
        std::vector<std::thread> pool;  // the pool is busy: threads of our own
        pool.reserve(threads - 1);
        for (unsigned t = 1; t < threads; ++t) pool.emplace_back([&] { job.drain(); });
        job.drain();
        for (auto& t : pool) t.join();
    }
    if (job.first) std::rethrow_exception(job.first);
}

}  // namespace foundry
