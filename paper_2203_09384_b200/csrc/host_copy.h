// Parallel host memcpy for the pageable-memory pipeline of sfft_execute_host.
//
// numpy arrays live in pageable memory; DMA from it goes through the driver's
// single-threaded bounce path (~6-13 GB/s measured).  Instead the host
// pipeline copies each chunk into pinned staging with several CPU threads and
// DMAs from there, overlapping the CPU copies of chunk c+1 with the PCIe
// transfers and kernel of chunk c.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace sfft_host {

class CopyPool {
 public:
  static CopyPool& instance() {
    static CopyPool pool;
    return pool;
  }

  // memcpy split into `workers() + 1` contiguous pieces (the caller copies one).
  void memcpy(void* dst, const void* src, size_t bytes) {
    const size_t kMinPiece = size_t(1) << 20;
    const int pieces = int(std::min<size_t>(threads_.size() + 1, std::max<size_t>(1, bytes / kMinPiece)));
    if (pieces <= 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const size_t step = (bytes + pieces - 1) / pieces;
    auto piece = [=](int i) {
      const size_t lo = size_t(i) * step;
      if (lo >= bytes) return;
      const size_t n = std::min(step, bytes - lo);
      std::memcpy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, n);
    };
    run(pieces, piece);
  }

  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }

 private:
  CopyPool() {
    // min(hardware threads / processes on this node, 16); SFFT_COPY_THREADS
    // overrides.  Measured on the 16-core B200 host, 512 MiB each way:
    // 8 threads 25.4 ms, 16 threads 23.0 ms, 24 threads 27.0 ms (host memory
    // bandwidth is the wall).  Under torchrun every rank of the node runs its
    // own pool, so the host's threads are split between them
    // (LOCAL_WORLD_SIZE) instead of oversubscribed.
    const unsigned hw = std::thread::hardware_concurrency();
    unsigned procs = 1;
    if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) {
      const int v = std::atoi(e);
      if (v >= 1 && v <= 1024) procs = unsigned(v);
    }
    unsigned want = std::min(std::max((hw ? hw : 1u) / procs, 1u), 16u);
    if (const char* e = std::getenv("SFFT_COPY_THREADS")) {
      const int v = std::atoi(e);
      if (v >= 1 && v <= 64) want = unsigned(v);
    }
    const int n = int(std::max(1u, want)) - 1;
    for (int i = 0; i < n; ++i) threads_.emplace_back([this, i] { loop(i + 1); });
  }

  // run fn(0..count-1): index 0 on the caller, the rest on the workers
  void run(int count, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> lk(call_mu_);  // one job at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &fn;
      count_ = count;
      pending_ = count - 1;
      ++generation_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

  void loop(int index) {
    unsigned long seen = 0;
    for (;;) {
      const std::function<void(int)>* job = nullptr;
      int count = 0;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || generation_ != seen; });
        if (stop_) return;
        seen = generation_;
        job = job_;
        count = count_;
      }
      if (job && index < count) {
        (*job)(index);
        std::lock_guard<std::mutex> g(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }

  std::vector<std::thread> threads_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int count_ = 0;
  int pending_ = 0;
  unsigned long generation_ = 0;
  bool stop_ = false;
};

}  // namespace sfft_host
