// A small persistent pool of host threads that splits a 2-D byte copy by
// rows (the pageable-buffer host entry stages user images through pinned
// bounce buffers; one memcpy thread cannot keep up with PCIe).
#pragma once

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace dctf {

class HostCopyPool {
 public:
  explicit HostCopyPool(int nthreads) : nparts_(nthreads < 1 ? 1 : nthreads) {
    for (int i = 1; i < nparts_; ++i) workers_.emplace_back([this, i] { run(i); });
  }
  ~HostCopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  HostCopyPool(const HostCopyPool&) = delete;
  HostCopyPool& operator=(const HostCopyPool&) = delete;

  // dst row r <- src row r (width bytes), r < rows; returns when all rows are copied
  void copy2d(uint8_t* dst, size_t dpitch, const uint8_t* src, size_t spitch, size_t width, int rows) {
    if (rows <= 0 || width == 0) return;
    {
      std::lock_guard<std::mutex> lk(mu_);
      task_ = Task{dst, dpitch, src, spitch, width, rows};
      pending_ = nparts_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    part(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  struct Task {
    uint8_t* dst;
    size_t dpitch;
    const uint8_t* src;
    size_t spitch, width;
    int rows;
  };
  void part(int k) {
    const Task t = task_;
    const int r0 = static_cast<int>(static_cast<long long>(t.rows) * k / nparts_);
    const int r1 = static_cast<int>(static_cast<long long>(t.rows) * (k + 1) / nparts_);
    if (t.dpitch == t.width && t.spitch == t.width)
      std::memcpy(t.dst + r0 * t.dpitch, t.src + r0 * t.spitch, static_cast<size_t>(r1 - r0) * t.width);
    else
      for (int r = r0; r < r1; ++r) std::memcpy(t.dst + r * t.dpitch, t.src + r * t.spitch, t.width);
  }
  void run(int k) {
    unsigned long long seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      lk.unlock();
      part(k);
      lk.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }

  const int nparts_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  Task task_{};
  int pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

}  // namespace dctf
