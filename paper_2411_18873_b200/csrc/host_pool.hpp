// Persistent host worker pool for the *_host entry points: the caller's Schedule[]
// rows are narrowed into pinned staging by all host cores while the GPU works on the
// previous chunk (the DMA then moves 24 instead of 96 bytes per candidate).
//
// One host_pipeline call runs ~16 jobs a few hundred microseconds apart (narrow chunk i, copy
// chunk i-2's outputs out).  A worker that finished a job spins on the job counter for a short
// while before it sleeps on the condition variable, so the next job of the same call starts
// without a futex wake-up per worker (measured: ~20 us per job with sleeping workers); between
// calls the workers sleep.
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__x86_64__) || defined(__i386__)
#include <immintrin.h>
#define ETUNE_POOL_PAUSE() _mm_pause()
#else
#define ETUNE_POOL_PAUSE() std::this_thread::yield()
#endif

namespace etune_b200 {

class HostPool {
public:
    explicit HostPool(int workers) {
        for (int i = 0; i < workers; ++i) threads_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_.store(true);
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    int size() const { return int(threads_.size()) + 1; }

    // fn(task) for task in [0, tasks), on the workers and the calling thread; returns
    // when every task has finished.  One run at a time (the ctx is single-threaded).
    void run(int tasks, const std::function<void(int)>& fn) {
        start(tasks, fn);
        join();
    }
    // run() in two halves: the workers begin at once, the caller may do other work (CUDA launches)
    // before it joins; fn must stay alive until join() returns.
    void start(int tasks, const std::function<void(int)>& fn) {
        if (tasks <= 0) {
            fn_ = nullptr;
            left_.store(0);
            return;
        }
        {
            std::lock_guard<std::mutex> g(mu_);
            fn_ = &fn;
            tasks_ = tasks;
            next_.store(0);
            left_.store(tasks);
            gen_.fetch_add(1, std::memory_order_release);  // publishes fn_ / tasks_ to spinning workers
        }
        if (sleepers_.load() > 0) cv_.notify_all();
    }
    void join() {
        if (fn_) work();
        while (left_.load(std::memory_order_acquire) != 0) ETUNE_POOL_PAUSE();
        fn_ = nullptr;
    }

private:
    static constexpr std::chrono::microseconds kSpin{300};

    void work() {
        for (;;) {
            const int t = next_.fetch_add(1);
            if (t >= tasks_) return;
            (*fn_)(t);
            left_.fetch_sub(1, std::memory_order_release);
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            // spin for the next job of the same call, then sleep
            const auto t0 = std::chrono::steady_clock::now();
            bool got = false;
            for (int it = 0;; ++it) {
                if (stop_.load()) return;
                if (gen_.load(std::memory_order_acquire) != seen) {
                    got = true;
                    break;
                }
                ETUNE_POOL_PAUSE();
                if ((it & 255) == 255 && std::chrono::steady_clock::now() - t0 > kSpin) break;
            }
            if (!got) {
                std::unique_lock<std::mutex> g(mu_);
                sleepers_.fetch_add(1);
                cv_.wait(g, [&] { return stop_.load() || gen_.load() != seen; });
                sleepers_.fetch_sub(1);
                if (stop_.load()) return;
            }
            {
                std::lock_guard<std::mutex> g(mu_);  // fn_ / tasks_ of the generation just seen
                seen = gen_.load();
            }
            work();
        }
    }

    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_;
    const std::function<void(int)>* fn_ = nullptr;
    int tasks_ = 0;
    std::atomic<int> next_{0}, left_{0}, sleepers_{0};
    std::atomic<uint64_t> gen_{0};
    std::atomic<bool> stop_{false};
};

}  // namespace etune_b200
