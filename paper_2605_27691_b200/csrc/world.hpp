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

// The refine phase's view of the transport (RankWorld's operations).
class World {
 public:
  virtual ~World() = default;
  virtual size_t num_ranks() const = 0;
  virtual void publish(size_t rank, const std::string& name, const void* dev_ptr, uint64_t bytes,
                       uint64_t wire_bytes, Runner& r) = 0;
  // Copies the target's current snapshot into dst (on r's device/stream).
  virtual uint64_t get(size_t src, size_t target, const std::string& name, void* dst,
                       Runner& r) = 0;
  virtual void barrier(size_t rank, Runner& r) = 0;
  virtual void abort(const std::string& reason) = 0;
  virtual std::vector<GetRecord> comm_log() const = 0;
};

// All ranks are host threads of this process (run_ranks, distsim.hpp:113-198).
class ThreadWorld : public World {
 public:
  ThreadWorld(size_t num_ranks, std::chrono::milliseconds watchdog = std::chrono::seconds(600),
              uint64_t epoch0 = 0);
  ~ThreadWorld() override;

  size_t num_ranks() const override { return num_ranks_; }
  uint64_t epoch() const;

  void publish(size_t rank, const std::string& name, const void* dev_ptr, uint64_t bytes,
               uint64_t wire_bytes, Runner& r) override;
  uint64_t get(size_t src, size_t target, const std::string& name, void* dst,
               Runner& r) override;
  uint64_t region_bytes(size_t target, const std::string& name);
  void barrier(size_t rank, Runner& r) override;
  void abort(const std::string& reason) override;
  bool aborted() const;
  std::vector<GetRecord> comm_log() const override;

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

// One rank per process (one process per GPU, e.g. torchrun).  Regions live in
// this process's device buffers; at every barrier the ranks all-gather their
// tables of current regions (name, CUDA IPC handle, sizes) through the host
// transport the caller supplies, and a get maps the target's buffer once
// (cudaIpcOpenMemHandle, cached) and pulls it with a device-to-device copy over
// NVLink.  A region becomes visible to other ranks at the next barrier -- the
// refine phase only reads regions after the barrier that follows their
// publish, so this matches RankWorld for the reference's schedule.
// Failure handling as RankWorld's (distsim.cpp:84-104): every exchange runs
// under a watchdog (KNNG_WORLD_WATCHDOG_S, default 600 s) -> WorldError, and a
// rank that fails aborts the world through its next exchange -> WorldAborted
// in every peer.
struct HostTransport {
  void* user = nullptr;
  // out = num_ranks consecutive blocks of `bytes`, in rank order; 0 = success
  int (*allgather)(void* user, const void* in, uint64_t bytes, void* out) = nullptr;
};

class ProcWorld : public World {
 public:
  ProcWorld(size_t num_ranks, size_t rank, const HostTransport& t);
  ~ProcWorld() override;

  size_t num_ranks() const override { return num_ranks_; }
  void publish(size_t rank, const std::string& name, const void* dev_ptr, uint64_t bytes,
               uint64_t wire_bytes, Runner& r) override;
  uint64_t get(size_t src, size_t target, const std::string& name, void* dst,
               Runner& r) override;
  void barrier(size_t rank, Runner& r) override;
  void abort(const std::string& reason) override;
  std::vector<GetRecord> comm_log() const override { return log_; }
  // all ranks' gets (collective: every rank must call it)
  std::vector<GetRecord> gather_comm_log();

  static constexpr int kMaxRegions = 8;
  // per-rank control word of every barrier exchange: an aborting rank's last
  // collective carries aborted = 1 and its reason, so peers waiting in that
  // barrier throw WorldAborted (distsim.cpp:96-104); epochs must agree
  // (mismatched barrier counts are a WorldError, the watchdog's case)
  struct Control {
    uint64_t epoch;
    int32_t aborted, pad;
    char reason[112];
  };
  struct Entry {  // fixed-size record exchanged at barriers
    char name[24];
    unsigned char handle[64];  // cudaIpcMemHandle_t
    uint64_t bytes, wire, cap;
    int32_t dev, valid;
  };

 private:
  struct Buf {
    void* p = nullptr;
    uint64_t bytes = 0, cap = 0, wire = 0;
    int dev = 0;
  };
  struct Slot {
    Buf current, staged;
    bool has_current = false, has_staged = false;
    uint64_t last_epoch = ~0ull;
  };
  void allgather(const void* in, uint64_t bytes, void* out);
  void exchange_tables(int aborted, const std::string& reason);

  const size_t num_ranks_, rank_;
  std::chrono::milliseconds watchdog_;
  HostTransport t_;
  std::map<std::string, Slot> mine_;
  std::vector<std::vector<Entry>> remote_;  // [rank][region]
  std::vector<GetRecord> log_;
  uint64_t epoch_ = 0;
  bool aborted_ = false;
  bool transport_dead_ = false;  // a collective failed or timed out: no more exchanges
};

}  // namespace knng_b200
