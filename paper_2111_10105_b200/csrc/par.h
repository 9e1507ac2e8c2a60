// Static-chunked parallel loop on a persistent host thread pool (decode
// analysis / mesh building).  Creating threads per loop costs more than
// most of these loops, so the workers live for the process and sleep on a
// condition variable between jobs.  One job runs at a time; a caller that
// finds the pool busy (another thread's job) runs its loop serially.
#pragma once
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <thread>
#include <vector>

namespace dmcg {

class HostPool {
 public:
  static HostPool& get() {
    static HostPool* pool = new HostPool();  // never destroyed: workers outlive static dtors
    return *pool;
  }
  uint32_t size() const { return (uint32_t)workers_.size() + 1; }

  // Runs call(ctx, c) for c in [0, nchunks): chunk 0 on the caller.
  // Returns false (nothing run) if the pool is busy.
  bool run(uint32_t nchunks, void (*call)(void*, uint32_t), void* ctx) {
    std::unique_lock<std::mutex> busy(busy_, std::try_to_lock);
    if (!busy.owns_lock()) return false;
    {
      std::lock_guard<std::mutex> lk(mu_);
      call_ = call;
      ctx_ = ctx;
      nchunks_ = nchunks;
      pending_.store(nchunks - 1, std::memory_order_relaxed);
      ++gen_;
    }
    cv_.notify_all();
    call(ctx, 0);
    // wait for the workers' chunks
    for (int spin = 0; pending_.load(std::memory_order_acquire) != 0; ++spin) {
      if (spin < 2000) {
        std::this_thread::yield();
      } else {
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_.load(std::memory_order_acquire) == 0; });
      }
    }
    return true;
  }

 private:
  HostPool() {
    const uint32_t hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    for (uint32_t t = 1; t < hw; ++t) workers_.emplace_back([this, t] { loop(t); });
    for (auto& w : workers_) w.detach();
  }
  void loop(uint32_t id) {
    uint64_t seen = 0;
    for (;;) {
      void (*call)(void*, uint32_t);
      void* ctx;
      uint32_t nch;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        call = call_;
        ctx = ctx_;
        nch = nchunks_;
      }
      if (id < nch) {
        call(ctx, id);
        if (pending_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
          std::lock_guard<std::mutex> lk(mu_);
          done_.notify_all();
        }
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex busy_, mu_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  void (*call_)(void*, uint32_t) = nullptr;
  void* ctx_ = nullptr;
  uint32_t nchunks_ = 0;
  std::atomic<uint32_t> pending_{0};
};

inline uint32_t parallel_chunks(uint32_t N, uint32_t grain) {
  const uint32_t hw = HostPool::get().size();
  return std::max(1u, std::min(hw, N / std::max(1u, grain)));
}

// fn(begin, end, chunk) over [0, N) split into parallel_chunks(N, grain)
// contiguous chunks (chunk ids are < 16).
template <class Fn>
void parallel_for(uint32_t N, uint32_t grain, const Fn& fn) {
  const uint32_t nt = parallel_chunks(N, grain);
  struct Job {
    const Fn* fn;
    uint32_t N, nt;
  } job{&fn, N, nt};
  auto call = [](void* p, uint32_t c) {
    const Job& j = *static_cast<const Job*>(p);
    (*j.fn)((uint32_t)((uint64_t)j.N * c / j.nt), (uint32_t)((uint64_t)j.N * (c + 1) / j.nt), c);
  };
  if (nt <= 1 || !HostPool::get().run(nt, call, &job))
    for (uint32_t c = 0; c < nt; ++c) call(&job, c);
}

}  // namespace dmcg
