// world.cpp -- ThreadWorld: RankWorld semantics (distsim.cpp:24-95) over
// device buffers, one host thread per rank, pulls as NVLink peer copies.
#include "world.hpp"

#include <algorithm>
#include <utility>

namespace knng_b200 {

uint64_t wire_region_size(RegionKind kind, uint64_t rows, uint64_t cols, bool u8_elems) {
  const uint64_t header = 4 + 1 + 8 + 8 + 1;  // wire.hpp:19
  const uint64_t cells = rows * cols;
  switch (kind) {
    case RegionKind::dataset:
      return header + cells * (u8_elems ? 1 : 4);
    case RegionKind::knng:
    case RegionKind::result:
      return header + cells * 8;
    case RegionKind::sgraph:
      return header + cells * 4;
  }
  return header;
}

ThreadWorld::ThreadWorld(size_t num_ranks, std::chrono::milliseconds watchdog)
    : num_ranks_(num_ranks), watchdog_(watchdog) {
  require(num_ranks >= 1, "RankWorld: P must be >= 1");
}

ThreadWorld::~ThreadWorld() {
  for (auto& kv : store_) {
    free_buf(kv.second.current);
    free_buf(kv.second.staged);
  }
}

void ThreadWorld::free_buf(Buf& b) {
  if (b.p) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(b.dev);
    cudaFree(b.p);
    cudaSetDevice(cur);
  }
  b = Buf{};
}

uint64_t ThreadWorld::epoch() const {
  std::lock_guard<std::mutex> l(mu_);
  return epoch_;
}

bool ThreadWorld::aborted() const {
  std::lock_guard<std::mutex> l(mu_);
  return aborted_;
}

void ThreadWorld::throw_if_aborted() const {
  if (aborted_) throw WorldAborted("world aborted: " + reason_);
}

void ThreadWorld::publish(size_t rank, const std::string& name, const void* dev_ptr,
                          uint64_t bytes, uint64_t wire_bytes, Runner& r) {
  require(rank < num_ranks_, "RankWorld: rank out of range");
  r.sync();  // the payload is final (this rank's kernels done) before the lock
  std::lock_guard<std::mutex> l(mu_);
  throw_if_aborted();
  Slot& s = store_[{rank, name}];
  if (s.published_once && s.last_epoch == epoch_)
    throw WorldError("publish: region '" + name + "' already published by rank " +
                     std::to_string(rank) + " in epoch " + std::to_string(epoch_));
  Buf* target = s.has_current ? &s.staged : &s.current;
  if (target->p && (target->bytes < bytes || target->dev != r.device)) free_buf(*target);
  DeviceGuard g(r.device);
  if (!target->p && bytes) {
    KNNG_CUDA(cudaMalloc(&target->p, bytes));
    target->dev = r.device;
  }
  target->bytes = bytes;
  target->wire = wire_bytes;
  if (bytes) {
    // the snapshot (copy = transfer, distsim.cpp:58) is complete before the
    // region becomes visible
    KNNG_CUDA(cudaMemcpyAsync(target->p, dev_ptr, bytes, cudaMemcpyDeviceToDevice, r.stream));
    r.sync();
  }
  if (s.has_current) s.has_staged = true; else s.has_current = true;
  s.published_once = true;
  s.last_epoch = epoch_;
}

uint64_t ThreadWorld::region_bytes(size_t target, const std::string& name) {
  std::lock_guard<std::mutex> l(mu_);
  auto it = store_.find({target, name});
  if (it == store_.end() || !it->second.has_current)
    throw WorldError("one_sided_get: region '" + name + "' not published by rank " +
                     std::to_string(target));
  return it->second.current.bytes;
}

uint64_t ThreadWorld::get(size_t src, size_t target, const std::string& name, void* dst,
                          Runner& r) {
  require(src < num_ranks_ && target < num_ranks_, "RankWorld: rank out of range");
  Buf b;
  {
    std::lock_guard<std::mutex> l(mu_);
    throw_if_aborted();
    auto it = store_.find({target, name});
    if (it == store_.end() || !it->second.has_current)
      throw WorldError("one_sided_get: region '" + name + "' not published by rank " +
                       std::to_string(target));
    b = it->second.current;
    log_.push_back({src, target, name, b.wire, epoch_, b.bytes});
  }
  if (b.bytes) {
    DeviceGuard g(r.device);
    if (b.dev == r.device)
      KNNG_CUDA(cudaMemcpyAsync(dst, b.p, b.bytes, cudaMemcpyDeviceToDevice, r.stream));
    else
      KNNG_CUDA(cudaMemcpyPeerAsync(dst, r.device, b.p, b.dev, b.bytes, r.stream));
  }
  return b.bytes;
}

void ThreadWorld::barrier(size_t rank, Runner& r) {
  require(rank < num_ranks_, "RankWorld: rank out of range");
  r.sync();  // this rank's pulls and publishes are complete
  std::unique_lock<std::mutex> l(mu_);
  throw_if_aborted();
  const uint64_t gen = generation_;
  if (++arrived_ == num_ranks_) {
    for (auto& kv : store_) {
      Slot& s = kv.second;
      if (s.has_staged) {
        std::swap(s.current, s.staged);  // old snapshot buffer is reused
        s.has_staged = false;
      }
    }
    ++epoch_;
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
    return;
  }
  const bool done =
      cv_.wait_for(l, watchdog_, [&] { return generation_ != gen || aborted_; });
  throw_if_aborted();
  if (!done) {
    aborted_ = true;
    reason_ = "barrier watchdog timeout at rank " + std::to_string(rank);
    cv_.notify_all();
    throw WorldError(reason_);
  }
}

void ThreadWorld::abort(const std::string& reason) {
  std::lock_guard<std::mutex> l(mu_);
  if (!aborted_) {
    aborted_ = true;
    reason_ = reason;
  }
  cv_.notify_all();
}

std::vector<GetRecord> ThreadWorld::comm_log() const {
  std::lock_guard<std::mutex> l(mu_);
  return log_;
}

}  // namespace knng_b200
