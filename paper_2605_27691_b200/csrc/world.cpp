// world.cpp -- ThreadWorld: RankWorld semantics (distsim.cpp:24-95) over
// device buffers, one host thread per rank, pulls as NVLink peer copies.
#include "world.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>
#include <thread>
#include <condition_variable>
#include <memory>

namespace knng_b200 {

namespace {

// Region buffers outlive a ThreadWorld: cudaMalloc/cudaFree synchronise the
// device (and, with peer access on, its peers), so a build that allocated its
// snapshot regions afresh stalled behind the other GPUs' kernels.  Freed
// regions park here per device and are reused by best fit.
struct RegionCache {
  struct Entry {
    int dev;
    uint64_t bytes;
    void* p;
  };
  std::mutex mu;
  std::vector<Entry> free_list;
  // buffers ever exported through a CUDA IPC handle (ProcWorld): peers may
  // still hold a mapping of them, and freeing an allocation that another
  // process has mapped is undefined, so these are never returned to the
  // driver (they are reused by best fit build after build; their set is
  // bounded by the largest build's regions)
  std::vector<void*> exported;
  static constexpr uint64_t kMaxCachedPerDev = uint64_t{24} << 30;

  void* acquire(int dev, uint64_t bytes, uint64_t* got) {
    {
      std::lock_guard<std::mutex> l(mu);
      size_t best = free_list.size();
      for (size_t i = 0; i < free_list.size(); ++i) {
        const Entry& e = free_list[i];
        if (e.dev != dev || e.bytes < bytes || e.bytes > 2 * bytes + (64u << 20)) continue;
        if (best == free_list.size() || e.bytes < free_list[best].bytes) best = i;
      }
      if (best != free_list.size()) {
        void* p = free_list[best].p;
        *got = free_list[best].bytes;
        free_list.erase(free_list.begin() + (std::ptrdiff_t)best);
        return p;
      }
    }
    void* p = nullptr;
    const double t0 = trace_clock_ms();
    KNNG_CUDA(cudaMalloc(&p, bytes));
    if (slow_trace_on())
      std::fprintf(stderr, "[knng slow] t %.1f region cudaMalloc %llu MB on dev %d: %.1f ms\n",
                   trace_clock_ms(), (unsigned long long)(bytes >> 20), dev,
                   trace_clock_ms() - t0);
    *got = bytes;
    return p;
  }
  void release(int dev, uint64_t bytes, void* p) {
    std::vector<Entry> evict;
    {
      std::lock_guard<std::mutex> l(mu);
      free_list.push_back({dev, bytes, p});
      uint64_t total = 0;
      for (const Entry& e : free_list)
        if (e.dev == dev) total += e.bytes;
      // over the cap: drop the oldest entries of this device
      for (size_t i = 0; i < free_list.size() && total > kMaxCachedPerDev;) {
        const bool pinned_by_peers =
            std::find(exported.begin(), exported.end(), free_list[i].p) != exported.end();
        if (free_list[i].dev == dev && !pinned_by_peers) {
          total -= free_list[i].bytes;
          evict.push_back(free_list[i]);
          free_list.erase(free_list.begin() + (std::ptrdiff_t)i);
        } else {
          ++i;
        }
      }
    }
    for (const Entry& e : evict) {
      DeviceGuard g(e.dev);
      const double t0 = trace_clock_ms();
      cudaFree(e.p);
      if (slow_trace_on())
        std::fprintf(stderr, "[knng slow] t %.1f region cudaFree %llu MB: %.1f ms\n",
                     trace_clock_ms(), (unsigned long long)(e.bytes >> 20), trace_clock_ms() - t0);
    }
  }
};

void mark_exported(void* p);

RegionCache& region_cache() {
  static RegionCache* c = new RegionCache();  // process lifetime (freed by the driver at exit)
  return *c;
}

void mark_exported(void* p) {
  RegionCache& c = region_cache();
  std::lock_guard<std::mutex> l(c.mu);
  if (std::find(c.exported.begin(), c.exported.end(), p) == c.exported.end())
    c.exported.push_back(p);
}

// Imported IPC mappings, process-wide: the exporting ranks keep their region
// buffers in their RegionCache, so a handle stays valid across builds and is
// opened once (cudaIpcOpenMemHandle / Close cost milliseconds and synchronise).
struct IpcMaps {
  std::mutex mu;
  std::map<std::string, void*> open;  // (device, handle bytes) -> mapped pointer
  void* map(int dev, const unsigned char* handle) {
    std::string key(reinterpret_cast<const char*>(handle), 64);
    key.append(reinterpret_cast<const char*>(&dev), sizeof(dev));
    std::lock_guard<std::mutex> l(mu);
    auto it = open.find(key);
    if (it != open.end()) return it->second;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    DeviceGuard g(dev);
    const double t0 = trace_clock_ms();
    KNNG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    if (slow_trace_on())
      std::fprintf(stderr, "[knng slow] t %.1f ipc open on dev %d: %.1f ms (%zu maps)\n",
                   trace_clock_ms(), dev, trace_clock_ms() - t0, open.size() + 1);
    open[key] = p;
    return p;
  }
};

IpcMaps& ipc_maps() {
  static IpcMaps* m = new IpcMaps();
  return *m;
}

}  // namespace

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

ThreadWorld::ThreadWorld(size_t num_ranks, std::chrono::milliseconds watchdog, uint64_t epoch0)
    : num_ranks_(num_ranks), watchdog_(watchdog), epoch_(epoch0) {
  require(num_ranks >= 1, "RankWorld: P must be >= 1");
}

ThreadWorld::~ThreadWorld() {
  for (auto& kv : store_) {
    free_buf(kv.second.current);
    free_buf(kv.second.staged);
  }
}

void ThreadWorld::free_buf(Buf& b) {
  if (b.p) region_cache().release(b.dev, b.cap ? b.cap : b.bytes, b.p);
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
  const double tp = trace_clock_ms();
  r.sync();  // the payload is final (this rank's kernels done) before the lock
  std::lock_guard<std::mutex> l(mu_);
  throw_if_aborted();
  Slot& s = store_[{rank, name}];
  if (s.published_once && s.last_epoch == epoch_)
    throw WorldError("publish: region '" + name + "' already published by rank " +
                     std::to_string(rank) + " in epoch " + std::to_string(epoch_));
  Buf* target = s.has_current ? &s.staged : &s.current;
  if (target->p && (target->cap < bytes || target->dev != r.device)) free_buf(*target);
  DeviceGuard g(r.device);
  if (!target->p && bytes) {
    target->p = region_cache().acquire(r.device, bytes, &target->cap);
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
  if (slow_trace_on())
    std::fprintf(stderr, "[knng slow] t %.1f rank %zu publish %s %.1f ms\n", trace_clock_ms(), rank,
                 name.c_str(), trace_clock_ms() - tp);
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
  const double tb = trace_clock_ms();
  struct Done {
    size_t rank;
    double tb;
    ~Done() {
      if (slow_trace_on())
        std::fprintf(stderr, "[knng slow] t %.1f rank %zu barrier %.1f ms\n", trace_clock_ms(),
                     rank, trace_clock_ms() - tb);
    }
  } done_trace{rank, tb};
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

// ---------------------------------------------------------------------------
// ProcWorld
// ---------------------------------------------------------------------------
ProcWorld::ProcWorld(size_t num_ranks, size_t rank, const HostTransport& t)
    : num_ranks_(num_ranks), rank_(rank), watchdog_(std::chrono::seconds(600)), t_(t) {
  if (const char* v = std::getenv("KNNG_WORLD_WATCHDOG_S"))
    watchdog_ = std::chrono::milliseconds((long long)(std::atof(v) * 1000.0));
  require(num_ranks >= 1 && rank < num_ranks, "RankWorld: rank out of range");
  require(t.allgather != nullptr, "RankWorld: the process transport needs an allgather");
  remote_.assign(num_ranks, {});
}

ProcWorld::~ProcWorld() {
  for (auto& kv : mine_) {
    for (Buf* b : {&kv.second.current, &kv.second.staged})
      if (b->p) region_cache().release(b->dev, b->cap, b->p);
  }
}

// The caller's all-gather on a helper thread, waited on with the watchdog: a
// peer that never arrives (crashed, hung, mismatched barrier counts) turns into
// a WorldError here instead of a hang.  On a timeout the helper is left
// blocked in the transport (it owns its buffers) and the world is dead.
void ProcWorld::allgather(const void* in, uint64_t bytes, void* out) {
  if (transport_dead_) throw WorldAborted("RankWorld: aborted (transport closed)");
  struct Call {
    std::vector<unsigned char> in, out;
    int rc = -1;
    bool done = false;
    std::mutex mu;
    std::condition_variable cv;
  };
  auto c = std::make_shared<Call>();
  c->in.assign(static_cast<const unsigned char*>(in), static_cast<const unsigned char*>(in) + bytes);
  c->out.resize(bytes * num_ranks_);
  HostTransport t = t_;
  std::thread([c, t] {
    const int rc = t.allgather(t.user, c->in.data(), c->in.size(), c->out.data());
    std::lock_guard<std::mutex> l(c->mu);
    c->rc = rc;
    c->done = true;
    c->cv.notify_all();
  }).detach();
  std::unique_lock<std::mutex> l(c->mu);
  if (!c->cv.wait_for(l, watchdog_, [&] { return c->done; })) {
    aborted_ = transport_dead_ = true;
    throw WorldError("barrier watchdog timeout at rank " + std::to_string(rank_));
  }
  if (c->rc != 0) {
    aborted_ = transport_dead_ = true;
    throw WorldAborted("RankWorld: host transport failed (another rank aborted?)");
  }
  std::memcpy(out, c->out.data(), c->out.size());
}

void ProcWorld::publish(size_t rank, const std::string& name, const void* dev_ptr,
                        uint64_t bytes, uint64_t wire_bytes, Runner& r) {
  require(rank == rank_, "RankWorld: a process publishes only its own rank's regions");
  require(name.size() < sizeof(Entry::name), "RankWorld: region name too long");
  if (aborted_) throw WorldAborted("RankWorld: aborted");
  r.sync();
  Slot& s = mine_[name];
  if (s.last_epoch == epoch_)
    throw WorldError("publish: region '" + name + "' already published by rank " +
                     std::to_string(rank) + " in epoch " + std::to_string(epoch_));
  Buf* target = s.has_current ? &s.staged : &s.current;
  if (target->p && (target->cap < bytes || target->dev != r.device)) {
    region_cache().release(target->dev, target->cap, target->p);
    *target = Buf{};
  }
  DeviceGuard g(r.device);
  if (!target->p && bytes) {
    target->p = region_cache().acquire(r.device, bytes, &target->cap);
    target->dev = r.device;
  }
  target->bytes = bytes;
  target->wire = wire_bytes;
  if (bytes) {
    KNNG_CUDA(cudaMemcpyAsync(target->p, dev_ptr, bytes, cudaMemcpyDeviceToDevice, r.stream));
    r.sync();
  }
  if (s.has_current) s.has_staged = true; else s.has_current = true;
  s.last_epoch = epoch_;
}

void ProcWorld::barrier(size_t rank, Runner& r) {
  require(rank == rank_, "RankWorld: rank out of range");
  if (aborted_) throw WorldAborted("RankWorld: aborted");
  r.sync();  // this rank's pulls and publishes are complete
  for (auto& kv : mine_) {
    Slot& s = kv.second;
    if (s.has_staged) {
      std::swap(s.current, s.staged);
      s.has_staged = false;
    }
  }
  ++epoch_;
  exchange_tables(0, std::string());
}

// One barrier exchange: Control + the tables of current regions, all-gathered
// (the all-gather is the barrier).
void ProcWorld::exchange_tables(int aborted, const std::string& reason) {
  constexpr size_t kBlock = sizeof(Control) + sizeof(Entry) * kMaxRegions;
  std::vector<unsigned char> blk(kBlock, 0);
  Control ctl{};
  ctl.epoch = epoch_;
  ctl.aborted = aborted;
  std::strncpy(ctl.reason, reason.c_str(), sizeof(ctl.reason) - 1);
  std::memcpy(blk.data(), &ctl, sizeof(ctl));
  std::vector<Entry> table(kMaxRegions);
  std::memset(table.data(), 0, sizeof(Entry) * kMaxRegions);
  int i = 0;
  for (auto& kv : mine_) {
    require(i < kMaxRegions, "RankWorld: too many regions");
    const Buf& b = kv.second.current;
    Entry& e = table[i++];
    std::strncpy(e.name, kv.first.c_str(), sizeof(e.name) - 1);
    e.bytes = b.bytes;
    e.wire = b.wire;
    e.cap = b.cap;
    e.dev = b.dev;
    e.valid = kv.second.has_current ? 1 : 0;
    if (b.p) {
      DeviceGuard g(b.dev);
      cudaIpcMemHandle_t h;
      KNNG_CUDA(cudaIpcGetMemHandle(&h, b.p));
      mark_exported(b.p);
      std::memcpy(e.handle, &h, sizeof(h));
    }
  }
  std::memcpy(blk.data() + sizeof(Control), table.data(), sizeof(Entry) * kMaxRegions);
  std::vector<unsigned char> all(kBlock * num_ranks_);
  allgather(blk.data(), kBlock, all.data());
  if (aborted) return;  // the abort notice is out; nothing more to learn
  for (size_t t = 0; t < num_ranks_; ++t) {
    Control pc;
    std::memcpy(&pc, all.data() + t * kBlock, sizeof(pc));
    if (pc.aborted) {
      aborted_ = transport_dead_ = true;
      pc.reason[sizeof(pc.reason) - 1] = 0;
      throw WorldAborted("world aborted: rank " + std::to_string(t) + ": " + pc.reason);
    }
    if (pc.epoch != epoch_) {
      aborted_ = transport_dead_ = true;
      throw WorldError("barrier: rank " + std::to_string(t) + " is at epoch " +
                       std::to_string(pc.epoch) + ", rank " + std::to_string(rank_) + " at " +
                       std::to_string(epoch_) + " (mismatched barrier counts)");
    }
    remote_[t].resize(kMaxRegions);
    std::memcpy(remote_[t].data(), all.data() + t * kBlock + sizeof(Control),
                sizeof(Entry) * kMaxRegions);
  }
}

uint64_t ProcWorld::get(size_t src, size_t target, const std::string& name, void* dst,
                        Runner& r) {
  require(src == rank_ && target < num_ranks_, "RankWorld: rank out of range");
  if (aborted_) throw WorldAborted("RankWorld: aborted");
  DeviceGuard g(r.device);
  if (target == rank_) {
    auto it = mine_.find(name);
    if (it == mine_.end() || !it->second.has_current)
      throw WorldError("one_sided_get: region '" + name + "' not published by rank " +
                       std::to_string(target));
    const Buf& b = it->second.current;
    log_.push_back({src, target, name, b.wire, epoch_, b.bytes});
    if (b.bytes)
      KNNG_CUDA(cudaMemcpyAsync(dst, b.p, b.bytes, cudaMemcpyDeviceToDevice, r.stream));
    return b.bytes;
  }
  const Entry* e = nullptr;
  for (const Entry& x : remote_[target])
    if (x.valid && name == x.name) e = &x;
  if (!e)
    throw WorldError("one_sided_get: region '" + name + "' not published by rank " +
                     std::to_string(target));
  log_.push_back({src, target, name, e->wire, epoch_, e->bytes});
  if (!e->bytes) return 0;
  void* p = ipc_maps().map(r.device, e->handle);
  // the owner runs nothing: a copy-engine pull over NVLink
  KNNG_CUDA(cudaMemcpyAsync(dst, p, e->bytes, cudaMemcpyDefault, r.stream));
  return e->bytes;
}

// RankWorld::abort: mark the world failed and tell the peers through one more
// exchange (their pending barrier all-gather receives it).  No-op once the
// world already failed or learned of a peer's abort.
void ProcWorld::abort(const std::string& reason) {
  if (aborted_) return;
  aborted_ = true;
  if (transport_dead_) return;
  try {
    exchange_tables(1, reason);
  } catch (...) {
  }
  transport_dead_ = true;
}

std::vector<GetRecord> ProcWorld::gather_comm_log() {
  struct Rec {
    uint64_t src, target, bytes, epoch, device_bytes;
    char region[24];
  };
  const uint64_t mine = log_.size();
  std::vector<uint64_t> counts(num_ranks_);
  allgather(&mine, sizeof(mine), counts.data());
  uint64_t mx = 0;
  for (uint64_t c : counts) mx = std::max(mx, c);
  std::vector<Rec> out(mx ? mx : 1), all((mx ? mx : 1) * num_ranks_);
  std::memset(out.data(), 0, sizeof(Rec) * out.size());
  for (uint64_t i = 0; i < mine; ++i) {
    const GetRecord& g = log_[i];
    out[i] = Rec{g.src, g.target, g.bytes, g.epoch, g.device_bytes, {0}};
    std::strncpy(out[i].region, g.region.c_str(), sizeof(out[i].region) - 1);
  }
  allgather(out.data(), sizeof(Rec) * out.size(), all.data());
  std::vector<GetRecord> res;
  for (size_t t = 0; t < num_ranks_; ++t)
    for (uint64_t i = 0; i < counts[t]; ++i) {
      const Rec& x = all[t * out.size() + i];
      res.push_back({x.src, x.target, x.region, x.bytes, x.epoch, x.device_bytes});
    }
  return res;
}

}  // namespace knng_b200
