// runtime.hpp -- host-side plumbing shared by the B200 kNN-graph library:
// error types mirroring the reference's exception classes, a per-(device,
// stream) Runner with stream-ordered allocations, and launch helpers.
#pragma once

#include <cuda_runtime.h>
#include <cstdlib>
#include <cstdio>
#include <chrono>

#include <mutex>
#include <thread>
#include <algorithm>
#include <utility>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"

namespace knng_b200 {

// Error classes map 1:1 onto the reference's:
//   std::invalid_argument (usage), WorldError/WorldAborted (transport),
//   FormatError (vecs/wire), std::logic_error (invariants).
struct WorldError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct WorldAborted : WorldError {
  using WorldError::WorldError;
};
struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void require(bool ok, const std::string& what) {
  if (!ok) throw std::invalid_argument(what);
}

// Device guard: sets the current device for the scope.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    KNNG_CUDA(cudaGetDevice(&prev));
    if (prev != dev) KNNG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// KNNG_TRACE_SLOW=1: host-side gaps > 30 ms between stage ticks, world ops.
inline bool slow_trace_on() {
  static const bool on = std::getenv("KNNG_TRACE_SLOW") != nullptr;
  return on;
}
inline double trace_clock_ms() {
  static const auto t0 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
inline int cur_device() {
  int d = -1;
  cudaGetDevice(&d);
  return d;
}

// One stream on one device.  All kernels of a call run on it, all temporaries
// are stream-ordered (cudaMallocAsync from the device pool, which we keep
// cached so steady-state iterations never hit the driver allocator).
struct Runner {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  bool owns = false;
  mutable cudaEvent_t sync_ev_ = nullptr;  // sync()'s event, created on first use

  Runner() = default;
  explicit Runner(int dev) : device(dev) {
    DeviceGuard g(dev);
    KNNG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    owns = true;
    KNNG_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
    cudaMemPool_t pool;
    KNNG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = ~0ull;
    KNNG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  // non-owning view of an existing stream (own scratch, the stream stays
  // with its owner)
  Runner(int dev, cudaStream_t s) : device(dev), stream(s), owns(false) {
    KNNG_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  Runner(const Runner&) = delete;
  Runner& operator=(const Runner&) = delete;
  Runner(Runner&& o) noexcept { *this = std::move(o); }
  Runner& operator=(Runner&& o) noexcept {
    device = o.device;
    stream = o.stream;
    num_sms = o.num_sms;
    owns = o.owns;
    scratch_ = std::move(o.scratch_);
    sync_ev_ = o.sync_ev_;
    o.sync_ev_ = nullptr;
    o.scratch_.clear();
    o.owns = false;
    o.stream = nullptr;
    return *this;
  }
  ~Runner() {
    if (stream) {
      cudaSetDevice(device);
      for (auto& sc : scratch_)
        if (sc.first) cudaFreeAsync(sc.first, stream);
    }
    if (owns && stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
    if (sync_ev_) cudaEventDestroy(sync_ev_);
  }
  // Wait for the stream by polling an event: a sleeping cudaStreamSynchronize
  // woke up late now and then (seen as idle GPU time of up to ~0.7 s per
  // build with four ranks per box).
  void sync() const {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != device) KNNG_CUDA(cudaSetDevice(device));
    if (!sync_ev_) KNNG_CUDA(cudaEventCreateWithFlags(&sync_ev_, cudaEventDisableTiming));
    KNNG_CUDA(cudaEventRecord(sync_ev_, stream));
    cudaError_t e;
    while ((e = cudaEventQuery(sync_ev_)) == cudaErrorNotReady) {
    }
    if (cur != device && cur >= 0) cudaSetDevice(cur);
    KNNG_CUDA(e);
  }

  // Grow-only stream-ordered scratch, one buffer per slot (kernels on this
  // stream that use a slot are ordered, so consecutive users share it).
  // Per-iteration temporaries come from here: allocating and freeing them
  // every iteration occasionally made the host wait on pool growth while
  // the GPU idled (up to ~55 ms, seen with KNNG_TRACE_SLOW).
  enum ScratchSlot {
    kScrScan = 0,
    kScrRadixHist,
    kScrRadixBase,
    kScrStage0,  // host datasets staged by a C-ABI call (two per call at most)
    kScrStage1,
    kScrCount
  };
  void* scratch(int slot, size_t bytes) const {
    if (scratch_.size() < (size_t)kScrCount) scratch_.resize(kScrCount, {nullptr, 0});
    auto& sc = scratch_[slot];
    if (sc.second < bytes) {
      DeviceGuard g(device);
      if (sc.first) cudaFreeAsync(sc.first, stream);
      const size_t cap = bytes + bytes / 4 + 256;
      KNNG_CUDA(cudaMallocAsync(&sc.first, cap, stream));
      sc.second = cap;
    }
    return sc.first;
  }

 private:
  mutable std::vector<std::pair<void*, size_t>> scratch_;
};

// Stream-ordered device buffer.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  int dev = 0;

  DBuf() = default;
  DBuf(const Runner& r, size_t count) { alloc(r, count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { swap(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    swap(o);
    return *this;
  }
  ~DBuf() { release(); }

  void swap(DBuf& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(s, o.s);
    std::swap(dev, o.dev);
  }
  void alloc(const Runner& r, size_t count) {
    release();
    s = r.stream;
    dev = r.device;
    n = count;
    if (count) {
      DeviceGuard g(dev);
      const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s);
      if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        throw CudaError(std::string("cudaMallocAsync of ") + std::to_string(count * sizeof(T)) +
                        " bytes on device " + std::to_string(dev) + " failed: " +
                        cudaGetErrorString(e) + " (free " + std::to_string(fr >> 20) + " MiB)");
      }
    }
  }
  void release() noexcept {
    if (p) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (cur != dev) cudaSetDevice(dev);
      cudaFreeAsync(p, s);
      if (cur != dev && cur >= 0) cudaSetDevice(cur);
    }
    p = nullptr;
    n = 0;
  }
  void zero() {
    if (n) KNNG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void fill_bytes(int v) {
    if (n) KNNG_CUDA(cudaMemsetAsync(p, v, n * sizeof(T), s));
  }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

// Pinned host scratch from a process-wide free list.  cudaFreeHost waits on
// every device and holds the driver while it does: a build_distributed whose
// ranks each freed a 64-byte counter buffer at the end of NN-descent measured
// stalls of up to 2.9 s (and the other GPUs' frees queued behind it).  Blocks
// are never returned to the driver.
struct PinnedPool {
  static void* get(size_t bytes, size_t* got) {
    PinnedPool& P = inst();
    {
      std::lock_guard<std::mutex> l(P.mu);
      for (size_t i = 0; i < P.free_list.size(); ++i) {
        if (P.free_list[i].second >= bytes) {
          void* p = P.free_list[i].first;
          *got = P.free_list[i].second;
          P.free_list.erase(P.free_list.begin() + (std::ptrdiff_t)i);
          return p;
        }
      }
    }
    const size_t cap = std::max<size_t>(bytes, 4096);
    void* p = nullptr;
    KNNG_CUDA(cudaMallocHost(&p, cap));
    *got = cap;
    return p;
  }
  static void put(void* p, size_t bytes) {
    PinnedPool& P = inst();
    std::lock_guard<std::mutex> l(P.mu);
    P.free_list.emplace_back(p, bytes);
  }

 private:
  static PinnedPool& inst() {
    static PinnedPool* p = new PinnedPool();  // process lifetime
    return *p;
  }
  std::mutex mu;
  std::vector<std::pair<void*, size_t>> free_list;
};

template <class T>
struct HBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t cap = 0;
  HBuf() = default;
  explicit HBuf(size_t count) { alloc(count); }
  HBuf(const HBuf&) = delete;
  HBuf& operator=(const HBuf&) = delete;
  ~HBuf() { release(); }
  void release() {
    if (p) PinnedPool::put(p, cap);
    p = nullptr;
    n = cap = 0;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(PinnedPool::get(count * sizeof(T), &cap));
  }
};

// memcpy into pageable memory split over threads: first-touch page faults of
// a fresh destination (e.g. np.empty) bound a single thread to ~5 GB/s.
inline void par_memcpy(char* dst, const char* src, size_t bytes) {
  constexpr int kThreads = 8;
  if (bytes < (size_t{4} << 20)) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t part = (bytes + kThreads - 1) / kThreads;
  std::thread t[kThreads - 1];
  for (int i = 1; i < kThreads; ++i) {
    const size_t lo = std::min(bytes, part * i), hi = std::min(bytes, part * (i + 1));
    t[i - 1] = std::thread([=] { std::memcpy(dst + lo, src + lo, hi - lo); });
  }
  std::memcpy(dst, src, std::min(bytes, part));
  for (auto& th : t) th.join();
}

// Device -> pageable host, synchronous: 16 MB chunks through two pinned pool
// buffers, the copy of chunk i overlapping the host memcpy of chunk i - 1
// (a direct copy into pageable memory measured ~4 GB/s).  Pinned
// destinations take the direct path.
inline void d2h_host(const Runner& r, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  cudaPointerAttributes at{};
  const bool pinned =
      cudaPointerGetAttributes(&at, dst) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  constexpr size_t kChunk = size_t{16} << 20;
  if (pinned || bytes <= kChunk) {
    KNNG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, r.stream));
    r.sync();
    return;
  }
  HBuf<char> buf[2];
  buf[0].alloc(kChunk);
  buf[1].alloc(kChunk);
  cudaEvent_t ev[2];
  KNNG_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  KNNG_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  size_t prev_off = 0, prev_len = 0;
  int i = 0;
  for (size_t off = 0; off < bytes; off += kChunk, ++i) {
    const size_t len = std::min(kChunk, bytes - off);
    KNNG_CUDA(cudaMemcpyAsync(buf[i & 1].p, s + off, len, cudaMemcpyDeviceToHost, r.stream));
    KNNG_CUDA(cudaEventRecord(ev[i & 1], r.stream));
    if (i > 0) {
      KNNG_CUDA(cudaEventSynchronize(ev[(i - 1) & 1]));
      par_memcpy(d + prev_off, buf[(i - 1) & 1].p, prev_len);
    }
    prev_off = off;
    prev_len = len;
  }
  KNNG_CUDA(cudaEventSynchronize(ev[(i - 1) & 1]));
  par_memcpy(d + prev_off, buf[(i - 1) & 1].p, prev_len);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
}

// Grid of persistent CTAs: `per_sm` resident CTAs on every SM.
inline unsigned persistent_grid(const Runner& r, int per_sm, uint64_t work_items) {
  uint64_t g = (uint64_t)r.num_sms * (uint64_t)per_sm;
  if (work_items < g) g = work_items ? work_items : 1;
  return (unsigned)g;
}

// Device-time breakdown by stage: tick(stage) records an event on the stream
// and attributes the interval since the previous tick to `stage`.
struct StageTimer {
  double last_host_ms = 0;
  bool on = false;
  cudaStream_t stream = nullptr;
  std::vector<cudaEvent_t> events;
  std::vector<int> stage_of;
  explicit StageTimer(bool enable, cudaStream_t s) : on(enable), stream(s) {
    if (on) tick(-1);
  }
  StageTimer(const StageTimer&) = delete;
  StageTimer& operator=(const StageTimer&) = delete;
  ~StageTimer() {
    for (auto e : events) cudaEventDestroy(e);
  }
  void tick(int stage) {
    if (slow_trace_on()) {
      const double t = trace_clock_ms();
      if (last_host_ms > 0 && t - last_host_ms > 30.0)
        std::fprintf(stderr, "[knng slow] t %.1f dev %d stage %d host %.1f ms\n", t,
                     cur_device(), stage, t - last_host_ms);
      last_host_ms = t;
    }
    if (!on) return;
    cudaEvent_t e;
    KNNG_CUDA(cudaEventCreate(&e));
    KNNG_CUDA(cudaEventRecord(e, stream));
    events.push_back(e);
    stage_of.push_back(stage);
  }
  // per-stage sums in ms (stream must be drained)
  void accumulate(double* out, int nstages) const {
    for (size_t i = 1; i < events.size(); ++i) {
      float ms = 0;
      KNNG_CUDA(cudaEventElapsedTime(&ms, events[i - 1], events[i]));
      if (stage_of[i] >= 0 && stage_of[i] < nstages) out[stage_of[i]] += ms;
    }
  }
  double total_ms() const {
    if (events.size() < 2) return 0.0;
    float ms = 0;
    KNNG_CUDA(cudaEventElapsedTime(&ms, events.front(), events.back()));
    return ms;
  }
};

// Prefix sum (scan.cu): out[0..n] exclusive scan of in[0..n), out[n] = total.
void exclusive_scan_u32(const Runner& r, const uint32_t* in, uint64_t* out, uint64_t n);

}  // namespace knng_b200
