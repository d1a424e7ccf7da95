// Host-side helpers for the slow-tier staging (emb.cu / uvm_cache.cuh):
//   ThreadPool   persistent threads for parallel_for (row gathers / scatters
//                between the pinned host tier and the pinned bounce buffers)
//   TaskQueue    one FIFO worker thread; tasks are numbered, callers can wait
//                for a task to finish; the first exception is kept and
//                rethrown to the caller at the next wait
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace rs {

class ThreadPool {
 public:
  explicit ThreadPool(unsigned n) {
    n = std::max(1u, n);
    for (unsigned i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~ThreadPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  unsigned size() const { return unsigned(th_.size()); }
  // fn(begin, end) over [0, n) split into contiguous ranges, one per thread
  void parallel_for(size_t n, const std::function<void(size_t, size_t)>& fn) {
    if (n == 0) return;
    std::unique_lock<std::mutex> g(mu_);
    job_ = &fn;
    n_ = n;
    left_ = unsigned(th_.size());
    ++epoch_;
    cv_.notify_all();
    done_.wait(g, [this] { return left_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(unsigned i) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> g(mu_);
    while (true) {
      cv_.wait(g, [&] { return stop_ || epoch_ != seen; });
      if (stop_) return;
      seen = epoch_;
      const auto* fn = job_;
      const size_t n = n_, k = th_.size();
      g.unlock();
      const size_t b = n * i / k, e = n * (i + 1) / k;
      if (b < e) (*fn)(b, e);
      g.lock();
      if (--left_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(size_t, size_t)>* job_ = nullptr;
  size_t n_ = 0;
  unsigned left_ = 0;
  uint64_t epoch_ = 0;
  bool stop_ = false;
};

class TaskQueue {
 public:
  TaskQueue() : th_([this] { loop(); }) {}
  ~TaskQueue() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  // returns the task's sequence number
  uint64_t post(std::function<void()> fn) {
    std::lock_guard<std::mutex> g(mu_);
    q_.push_back(std::move(fn));
    cv_.notify_all();
    return ++posted_;
  }
  // blocks until task `seq` (and every earlier one) has run
  void wait(uint64_t seq) {
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return done_ >= seq; });
    rethrow_locked();
  }
  void drain() { wait(posted()); }
  uint64_t posted() {
    std::lock_guard<std::mutex> g(mu_);
    return posted_;
  }

 private:
  void rethrow_locked() {
    if (err_) {
      auto e = err_;
      err_ = nullptr;
      std::rethrow_exception(e);
    }
  }
  void loop() {
    std::unique_lock<std::mutex> g(mu_);
    while (true) {
      cv_.wait(g, [&] { return stop_ || !q_.empty(); });
      if (q_.empty() && stop_) return;
      auto fn = std::move(q_.front());
      q_.pop_front();
      g.unlock();
      try {
        fn();
      } catch (...) {
        std::lock_guard<std::mutex> g2(mu_);
        if (!err_) err_ = std::current_exception();
      }
      g.lock();
      ++done_;
      done_cv_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<std::function<void()>> q_;
  uint64_t posted_ = 0, done_ = 0;
  bool stop_ = false;
  std::exception_ptr err_;
  std::thread th_;  // last: starts after the members above exist
};

}  // namespace rs
