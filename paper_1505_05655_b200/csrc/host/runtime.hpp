// runtime.hpp -- device context of the B200 backend: bound devices, per-device
// pools of request slots (stream + device buffers + pinned staging), and the
// host<->HBM staging helpers.
//
// This replaces the reference's payload staging, where every request lands
// in a zero-filled pageable std::vector (proj/src/server.cpp:95-101) and is
// copied again by the codec (proj/src/demosaic.cpp:177-209) and the response
// framing (proj/src/registry.cpp:129).  Here a request's bytes go host ->
// HBM once, with async copies on the slot's own stream; pageable callers are
// staged through double-buffered pinned chunks so the memcpy of chunk i
// overlaps the DMA of chunk i-1.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../../include/gpcx.h"
#include "../kernels.hpp"

namespace gpcx::rt {

// Grow-only device allocation.
struct DeviceBuf {
  void* ptr = nullptr;
  std::uint64_t cap = 0;
  void ensure(std::uint64_t bytes, bool zero = false);
  void release();
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

struct PinnedBuf {
  void* ptr = nullptr;
  std::uint64_t cap = 0;
  void ensure(std::uint64_t bytes);
  void release();
};

inline constexpr std::uint64_t kStageChunk = 8ull << 20;

// Everything one in-flight request needs on one device.
struct Slot {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t chunk_done[2] = {nullptr, nullptr};
  cudaEvent_t ready = nullptr;  // cross-device handoff (e.g. a staged B slice)
  DeviceBuf a, b, c;     // operands / result
  DeviceBuf lut_ws;      // LUT workspace (zeroed once, self-cleaning)
  DeviceBuf mm_ws;       // tensor-core matmul workspace
  DeviceBuf small;       // LUT (128 KiB) + stats + hist
  PinnedBuf stage[2];    // pageable-caller staging chunks
  PinnedBuf h_small;     // stats readback
  std::uint16_t* d_lut() const { return small.as<std::uint16_t>(); }
  gpcx_lut_stats* d_stats() const {
    return reinterpret_cast<gpcx_lut_stats*>(small.as<unsigned char>() + 131072);
  }
  std::uint32_t* d_hist() const {
    return reinterpret_cast<std::uint32_t*>(small.as<unsigned char>() + 131072 + 256);
  }
  // device copy of the band's PeerTable (the in-process LUT exchange)
  lut::PeerTable* d_peer_table() const {
    return reinterpret_cast<lut::PeerTable*>(small.as<unsigned char>() + 131072 + 256 +
                                             65536 * 4);
  }
  gpcx_lut_stats* h_stats() const { return static_cast<gpcx_lut_stats*>(h_small.ptr); }
  // u64 digest scratch next to the stats (device) / in the readback buffer
  std::uint64_t* d_digest() const {
    return reinterpret_cast<std::uint64_t*>(small.as<unsigned char>() + 131072 + 128);
  }
  std::uint64_t* h_digest() const {
    return reinterpret_cast<std::uint64_t*>(static_cast<unsigned char*>(h_small.ptr) + 128);
  }
  ~Slot();
};

class Runtime;

// RAII lease of a slot; returns it to its device pool.
class SlotLease {
 public:
  SlotLease(Runtime* rt, Slot* slot) : rt_(rt), slot_(slot) {}
  SlotLease(SlotLease&& o) noexcept : rt_(o.rt_), slot_(o.slot_) { o.slot_ = nullptr; }
  SlotLease(const SlotLease&) = delete;
  ~SlotLease();
  Slot* operator->() const { return slot_; }
  Slot& operator*() const { return *slot_; }

 private:
  Runtime* rt_;
  Slot* slot_;
};

// Thread-local device affinity: while alive, pick_device_index() on this
// thread returns `index` (the server's per-device workers), as long as that
// device is healthy.
class Affinity {
 public:
  explicit Affinity(int index);
  ~Affinity();
  Affinity(const Affinity&) = delete;
  Affinity& operator=(const Affinity&) = delete;

 private:
  int saved_;
};

// Device health (SURVEY.md §5 failure detection; the reference's failure
// boundary is the handler exception -> ERR:TASK_FAILED, proj/src/
// registry.cpp:113-118).  A sticky CUDA error (illegal address, launch
// failure, trap, ...) poisons the device's context for the whole process:
// every later call on it fails.  The runtime therefore QUARANTINES the
// device -- its idle slots are retired, leased ones are not returned, no new
// request is routed to it, the planner shards only over healthy devices --
// and requests keep running on the remaining ones; only when none is left
// does every GPU request answer ERR:TASK_FAILED ("no healthy device").  The
// request that hit the fault fails (it is not retried elsewhere: a fault its
// data caused would poison the next device too).  A quarantined device is
// not reset in-process (cudaDeviceReset would free pinned host buffers and
// peer mappings other devices' work still uses); rebinding with gpcx_init or
// restarting the server process brings it back.
bool is_sticky(cudaError_t e);
// Called on every failed CUDA call (GPCX_CUDA): quarantines the calling
// thread's current device when `e` is sticky.
void note_cuda_error(cudaError_t e, const char* where);

class Runtime {
 public:
  static Runtime& get();
  // devices empty -> all visible devices.  Rebinding to a different set
  // drains the pools first.
  void init(const std::vector<int>& devices);
  void shutdown();
  std::vector<int> devices();
  int ndev();
  // The thread's affinity if set and healthy, else round robin over the
  // healthy bound devices (C5 replicas); TaskFailed when none is healthy.
  int pick_device_index();
  std::vector<int> healthy_indices();
  bool healthy(int index);
  std::string health_reason(int index);  // "" while healthy
  void quarantine_device(int ordinal, const std::string& why);  // every index bound to it
  void quarantine_index(int index, const std::string& why);     // one bound index (tests)
  // Device ordinal of bound index i.
  int device_at(int index);
  SlotLease acquire(int device_index);
  void release(Slot* slot);

 private:
  struct Pool {
    int device;
    std::vector<std::unique_ptr<Slot>> all;
    std::vector<Slot*> free;
    bool healthy = true;
    std::string why;  // first sticky error seen on it
  };
  void retire_idle_locked(Pool& pool);
  void ensure_init_locked();
  std::mutex mu_;
  bool inited_ = false;
  std::vector<Pool> pools_;
  std::atomic<unsigned> rr_{0};
};

// A request payload still arriving from the network into a pinned buffer
// (SURVEY.md §8f row 2).  While it is registered, h2d() of a range inside
// it copies chunk by chunk as the bytes land, so the DMA to HBM overlaps
// the receive instead of starting after the last byte.
class Arrival {
 public:
  Arrival(const void* base, std::uint64_t len);
  ~Arrival();
  Arrival(const Arrival&) = delete;
  Arrival& operator=(const Arrival&) = delete;
  void advance(std::uint64_t got);  // bytes [0, got) are in place
  void fail();                      // the receive failed: waiters throw Truncated
  void wait_for(std::uint64_t upto);
  const std::uint8_t* base() const { return base_; }
  std::uint64_t size() const { return len_; }

 private:
  const std::uint8_t* base_;
  std::uint64_t len_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::uint64_t got_ = 0;
  bool failed_ = false;
};
inline constexpr std::uint64_t kArrivalChunk = 4ull << 20;

// Host -> device copy on the slot stream.  Pinned sources go straight to the
// DMA engine; pageable sources are staged chunk-wise (returns once the last
// chunk's memcpy is issued; the caller syncs the stream before reusing src).
void h2d(Slot& s, void* dst, const void* src, std::uint64_t bytes);
// Device -> host copy on the slot stream; synchronises before returning.
void d2h(Slot& s, void* dst, const void* src, std::uint64_t bytes);
bool is_pinned(const void* p);

// Pool of page-locked host buffers (cudaMallocHost costs ~ms per GiB, so
// request/response staging buffers are recycled by power-of-two size class).
class PinnedLease {
 public:
  PinnedLease() = default;
  PinnedLease(void* p, std::uint64_t cap, bool pageable = false)
      : ptr_(p), cap_(cap), pageable_(pageable) {}
  PinnedLease(PinnedLease&& o) noexcept : ptr_(o.ptr_), cap_(o.cap_), pageable_(o.pageable_) {
    o.ptr_ = nullptr;
  }
  PinnedLease& operator=(PinnedLease&& o) noexcept;
  PinnedLease(const PinnedLease&) = delete;
  ~PinnedLease();
  void* get() const { return ptr_; }
  std::uint64_t capacity() const { return cap_; }

 private:
  void* ptr_ = nullptr;
  std::uint64_t cap_ = 0;
  bool pageable_ = false;  // page-locking unavailable (no usable device)
};
// A pooled pinned buffer.  Page-locked bytes leased at once are bounded
// (GPCX_PINNED_CAP_MB, default 32 GiB): past the bound -- e.g. many clients
// that sent only headers of large requests -- a lease is plain heap memory,
// which the staging copies handle through their chunked pinned bounce
// buffers.  When page-locking fails (no usable device) also a heap buffer,
// so framing still works and the handler reports the GPU error.
PinnedLease pinned_acquire(std::uint64_t bytes);
std::uint64_t pinned_in_use();  // page-locked bytes currently leased
void pinned_trim();  // frees idle pooled buffers

// Makes `device` current for the calling thread.
void use_device(int device);
// true when `from` has peer access to `to`'s memory (or from == to).
bool peer_reachable(int from, int to);

}  // namespace gpcx::rt
