// world.hpp -- the transport boundary of the refine phase on B200s.
//
// Mirrors RankWorld (distsim.hpp:36-87, distsim.cpp:24-95) over device memory:
//   publish(rank, name, dev_ptr, bytes): a rank makes a device region visible.
//       First publish of a name is visible immediately; a republish is staged
//       and swapped in by the next barrier; one publish per name per epoch.
//       The payload is copied into a world-owned buffer on the publisher's GPU
//       (the snapshot; "copy = transfer" distsim.cpp:58).
//   get(src, target, name, dst): one-sided pull -- a cudaMemcpyPeerAsync over
//       NVLink from the target GPU's snapshot into the caller's buffer; the
//       target runs nothing.  Logged with the reference's wire byte count
//       (wire::region_size) so comm accounting matches acceptance.cpp:253-322.
//   barrier(rank): all ranks' streams drained, staged regions swapped, epoch++;
//       a watchdog converts a missing rank into WorldError (distsim.cpp:84-94).
//   abort(reason): wakes waiters, which throw WorldAborted.
#pragma once

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "runtime.hpp"

namespace knng_b200 {

struct GetRecord {
  uint64_t src = 0;
  uint64_t target = 0;
  std::string region;
  uint64_t bytes = 0;  // serialized (wire) size, as the reference logs
  uint64_t epoch = 0;
  uint64_t device_bytes = 0;  // bytes actually moved
};

// wire::region_size (wire.cpp:47-68): 22-byte header + payload.
enum class RegionKind : uint8_t { dataset = 0, knng = 1, sgraph = 2, result = 3 };
uint64_t wire_region_size(RegionKind kind, uint64_t rows, uint64_t cols, bool u8_elems = false);

class ThreadWorld {
 public:
  ThreadWorld(size_t num_ranks, std::chrono::milliseconds watchdog = std::chrono::seconds(600));
  ~ThreadWorld();

  size_t num_ranks() const { return num_ranks_; }
  uint64_t epoch() const;

  void publish(size_t rank, const std::string& name, const void* dev_ptr, uint64_t bytes,
               uint64_t wire_bytes, Runner& r);
  // Copies the target's current snapshot into dst (on r's device/stream).
  uint64_t get(size_t src, size_t target, const std::string& name, void* dst, Runner& r);
  uint64_t region_bytes(size_t target, const std::string& name);
  void barrier(size_t rank, Runner& r);
  void abort(const std::string& reason);
  bool aborted() const;
  std::vector<GetRecord> comm_log() const;

 private:
  struct Buf {
    void* p = nullptr;
    uint64_t bytes = 0;
    uint64_t cap = 0;  // allocation size (buffers come from a reuse cache)
    uint64_t wire = 0;
    int dev = 0;
  };
  struct Slot {
    Buf current, staged;
    bool has_current = false, has_staged = false;
    bool published_once = false;
    uint64_t last_epoch = 0;
  };
  static void free_buf(Buf& b);
  void throw_if_aborted() const;

  const size_t num_ranks_;
  const std::chrono::milliseconds watchdog_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::pair<size_t, std::string>, Slot> store_;
  std::vector<GetRecord> log_;
  uint64_t epoch_ = 0;
  uint64_t generation_ = 0;
  size_t arrived_ = 0;
  bool aborted_ = false;
  std::string reason_;
};

}  // namespace knng_b200
