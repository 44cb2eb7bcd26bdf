// The serial I/O channel of AsyncIO (simulator.cpp:181-227, rules R2/R7/R8) on real
// hardware: one copy stream owned by one host thread, a FIFO of expert copies with
// cancellable queued prefetches, at most `depth` copies enqueued on the copy stream
// (1 in the engine: issued = started, as R2 needs), and HBM slots whose
// reuse waits for the compute that last read them. Shared by the decode engine
// (engine.cpp) and the stand-alone expert cache (cache.cpp).
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "cuda_host.hpp"

namespace ps {

inline double io_now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Slot {
  void* dev = nullptr;
  void* zdev = nullptr;            // landing buffer of a z-slab copy (decoded into dev)
  cudaEvent_t free_ev = nullptr;   // recorded on the compute stream after the last reader
  std::atomic<int64_t> recorded_gen{0};
  int64_t next_gen = 0;            // generation a new copy must wait for
  bool in_use = false;
  int target_layer = -1;
};

enum JobKind { kOnDemand = 0, kPrefetch = 1 };

struct IoJob {
  int kind = kOnDemand;
  int layer = 0, expert = 0, tokens = 0;
  void* dst = nullptr;
  const void* src = nullptr;
  size_t bytes = 0;
  Slot* slot = nullptr;
  int64_t wait_gen = 0;        // slot->recorded_gen must reach this before issue
  cudaEvent_t start_ev = nullptr, done_ev = nullptr;
  std::atomic<int> state{0};   // 0 queued, 1 issued, 2 cancelled
  bool critical = false;
  int issue_group = 1;
  const uint8_t* zhost = nullptr;  // z-slab source (header read on the host), null = raw copy
  double t_io_us = 0;              // modelled transfer time (cost.t_io)
  std::atomic<double> est_done_us{0};  // host-clock estimate of the copy's end (set at issue)
};

// The serial I/O channel: one copy stream, one host thread, FIFO with cancel.
class IoChannel {
 public:
  IoChannel(int device, int depth) : depth_(depth) {
    device_ = device;
    PS_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    thread_ = std::thread([this] { run(); });
  }
  ~IoChannel() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    thread_.join();
    cudaStreamDestroy(stream_);
  }
  cudaStream_t stream() const { return stream_; }

  void push(IoJob* j) {
    {
      std::lock_guard<std::mutex> g(mu_);
      queue_.push_back(j);
    }
    cv_.notify_all();
  }
  // Ahead of every queued (not yet issued) job: an on-demand load overtakes queued
  // prefetches (R7 before R8); copies already issued run to completion.
  void push_front(IoJob* j) {
    {
      std::lock_guard<std::mutex> g(mu_);
      queue_.push_front(j);
    }
    cv_.notify_all();
  }
  void notify() { cv_.notify_all(); }
  void wait_issued(IoJob* j) {
    std::unique_lock<std::mutex> g(mu_);
    cv_.wait(g, [&] { return j->state.load() != 0 || error_; });
    if (error_) fail(PS_ECUDA, "I/O channel: " + err_msg_);
  }
  // Cancel queued (not yet issued) prefetch jobs; returns them (R2).
  std::vector<IoJob*> cancel_queued_prefetches() {
    std::vector<IoJob*> out;
    std::lock_guard<std::mutex> g(mu_);
    for (auto it = queue_.begin(); it != queue_.end();) {
      if ((*it)->kind == kPrefetch && (*it)->state.load() == 0) {
        (*it)->state = 2;
        out.push_back(*it);
        it = queue_.erase(it);
      } else {
        ++it;
      }
    }
    return out;
  }
  // Step entry after a failed step: forget every job still queued (their FFNs were never
  // launched, so slot generations they wait for would never come).
  void abandon_queued() {
    std::lock_guard<std::mutex> g(mu_);
    for (IoJob* j : queue_) j->state = 2;
    queue_.clear();
    cv_.notify_all();
  }
  void drain() {  // wait until the queue is empty and every issued copy completed
    std::unique_lock<std::mutex> g(mu_);
    cv_.wait(g, [&] { return (queue_.empty() && !busy_) || error_; });
    g.unlock();
    PS_CUDA(cudaStreamSynchronize(stream_));
  }
  void check() {
    std::lock_guard<std::mutex> g(mu_);
    if (error_) fail(PS_ECUDA, "I/O channel: " + err_msg_);
  }

 private:
  void run() {
    cudaSetDevice(device_);
    std::deque<cudaEvent_t> in_flight;
    std::unique_lock<std::mutex> g(mu_);
    while (true) {
      cv_.wait(g, [&] { return stop_ || !queue_.empty(); });
      if (stop_) break;
      busy_ = true;
      // Throttle: at most depth_ copies in flight, so later queue entries stay
      // cancellable until the channel is about to free up. An on-demand load is never
      // cancelled, so it may always be enqueued behind one running copy (back-to-back
      // loads keep the link busy); the limit applies to prefetches.
      auto limit = [&] { return !queue_.empty() && queue_.front()->kind == kOnDemand ? std::max(depth_, 2) : depth_; };
      while (static_cast<int>(in_flight.size()) >= limit()) {
        cudaEvent_t ev = in_flight.front();
        g.unlock();
        cudaError_t e = cudaEventSynchronize(ev);
        g.lock();
        in_flight.pop_front();
        if (e != cudaSuccess) set_error(e);
      }
      if (queue_.empty()) {
        busy_ = false;
        cv_.notify_all();
        continue;
      }
      IoJob* j = queue_.front();
      if (j->slot && j->slot->recorded_gen.load() < j->wait_gen) {
        // Slot still owned by an FFN the engine has not launched yet: wait for it.
        cv_.wait(g, [&] { return stop_ || j->slot->recorded_gen.load() >= j->wait_gen || queue_.empty() ||
                                 queue_.front() != j; });
        if (stop_) break;
        busy_ = false;
        cv_.notify_all();  // drain() may be waiting for busy_ to clear (abandoned queue)
        continue;  // re-evaluate the front (it may have been cancelled)
      }
      queue_.pop_front();
      g.unlock();
      cudaError_t e = cudaSuccess;
      if (j->slot && j->wait_gen > 0) e = cudaStreamWaitEvent(stream_, j->slot->free_ev, 0);
      if (e == cudaSuccess) e = cudaEventRecord(j->start_ev, stream_);
      if (e == cudaSuccess) e = cudaMemcpyAsync(j->dst, j->src, j->bytes, cudaMemcpyHostToDevice, stream_);
      if (e == cudaSuccess) e = cudaEventRecord(j->done_ev, stream_);
      // FIFO channel: this copy ends t_io after the later of now and the previous end
      est_end_ = std::max(est_end_, io_now_us()) + j->t_io_us;
      j->est_done_us.store(est_end_);
      g.lock();
      if (e != cudaSuccess) set_error(e);
      in_flight.push_back(j->done_ev);
      j->state = 1;
      busy_ = !queue_.empty();
      cv_.notify_all();
    }
  }
  void set_error(cudaError_t e) {
    error_ = true;
    err_msg_ = cudaGetErrorString(e);
    cv_.notify_all();
  }

  int device_ = 0;
  int depth_;
  cudaStream_t stream_ = nullptr;
  std::thread thread_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<IoJob*> queue_;
  double est_end_ = 0;  // modelled end of the last issued copy (I/O thread only)
  bool stop_ = false, busy_ = false, error_ = false;
  std::string err_msg_;
};

}  // namespace ps
