// Persistent host worker pool for the *_host entry points: the caller's Schedule[]
// rows are narrowed into pinned staging by all host cores while the GPU works on the
// previous chunk (the DMA then moves 24 instead of 96 bytes per candidate).
#pragma once

#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace etune_b200 {

class HostPool {
public:
    explicit HostPool(int workers) {
        for (int i = 0; i < workers; ++i) threads_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    int size() const { return int(threads_.size()) + 1; }

    // fn(task) for task in [0, tasks), on the workers and the calling thread; returns
    // when every task has finished.
    void run(int tasks, const std::function<void(int)>& fn) {
        if (tasks <= 0) return;
        {
            std::lock_guard<std::mutex> g(mu_);
            fn_ = &fn;
            tasks_ = tasks;
            next_.store(0);
            left_.store(tasks);
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(mu_);
        done_cv_.wait(g, [this] { return left_.load() == 0; });
        fn_ = nullptr;
    }

private:
    void work() {
        for (;;) {
            const int t = next_.fetch_add(1);
            if (t >= tasks_) return;
            (*fn_)(t);
            if (left_.fetch_sub(1) == 1) {
                std::lock_guard<std::mutex> g(mu_);
                done_cv_.notify_all();
            }
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }

    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    int tasks_ = 0;
    std::atomic<int> next_{0}, left_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

}  // namespace etune_b200
