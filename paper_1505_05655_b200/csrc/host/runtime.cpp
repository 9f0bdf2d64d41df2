// runtime.cpp -- see runtime.hpp.
#include "runtime.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>

#include "../cuda_util.hpp"
#include "../kernels.hpp"
#include "trace.hpp"

namespace gpcx::rt {

void use_device(int device) { GPCX_CUDA(cudaSetDevice(device)); }

namespace {
thread_local int t_affinity = -1;
}  // namespace

Affinity::Affinity(int index) : saved_(t_affinity) { t_affinity = index; }
Affinity::~Affinity() { t_affinity = saved_; }

bool is_sticky(cudaError_t e) {
  switch (e) {
    case cudaErrorIllegalAddress:
    case cudaErrorLaunchFailure:  // includes __trap()
    case cudaErrorIllegalInstruction:
    case cudaErrorMisalignedAddress:
    case cudaErrorInvalidAddressSpace:
    case cudaErrorInvalidPc:
    case cudaErrorHardwareStackError:
    case cudaErrorAssert:
    case cudaErrorLaunchTimeout:
    case cudaErrorECCUncorrectable:
    case cudaErrorContextIsDestroyed:
      return true;
    default:
      return false;
  }
}

void note_cuda_error(cudaError_t e, const char* where) {
  if (!is_sticky(e)) return;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return;
  Runtime::get().quarantine_device(
      dev, std::string(cudaGetErrorName(e)) + " at " + (where != nullptr ? where : "?"));
}

void DeviceBuf::ensure(std::uint64_t bytes, bool zero) {
  if (bytes <= cap && ptr != nullptr) return;
  release();
  const std::uint64_t want = std::max<std::uint64_t>(bytes, 256);
  GPCX_CUDA(cudaMalloc(&ptr, want));
  cap = want;
  if (zero) {
    // complete before any (non-blocking) stream uses the buffer
    GPCX_CUDA(cudaMemset(ptr, 0, want));
    GPCX_CUDA(cudaStreamSynchronize(nullptr));
  }
}

void DeviceBuf::release() {
  if (ptr != nullptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
}

void PinnedBuf::ensure(std::uint64_t bytes) {
  if (bytes <= cap && ptr != nullptr) return;
  release();
  GPCX_CUDA(cudaMallocHost(&ptr, std::max<std::uint64_t>(bytes, 256)));
  cap = std::max<std::uint64_t>(bytes, 256);
}

void PinnedBuf::release() {
  if (ptr != nullptr) cudaFreeHost(ptr);
  ptr = nullptr;
  cap = 0;
}

Slot::~Slot() {
  cudaSetDevice(device);
  if (stream != nullptr) cudaStreamSynchronize(stream);
  a.release();
  b.release();
  c.release();
  lut_ws.release();
  mm_ws.release();
  small.release();
  stage[0].release();
  stage[1].release();
  h_small.release();
  for (cudaEvent_t& e : chunk_done)
    if (e != nullptr) cudaEventDestroy(e);
  if (ready != nullptr) cudaEventDestroy(ready);
  if (stream != nullptr) cudaStreamDestroy(stream);
}

SlotLease::~SlotLease() {
  if (slot_ != nullptr) rt_->release(slot_);
}

Runtime& Runtime::get() {
  static Runtime* rt = new Runtime();  // never destroyed: outlives static teardown
  return *rt;
}

namespace {
// Direct NVLink access between every pair of bound devices, so a peer copy
// (cudaMemcpyPeerAsync) is one DMA over NVSwitch instead of a host bounce.
// Best effort: without it the copies still work, just staged.
std::mutex g_peer_mu;
std::set<std::pair<int, int>> g_peer_on;  // (d, p): d may load p's memory

void enable_peer_access(const std::vector<int>& devs) {
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return;
  std::lock_guard<std::mutex> lock(g_peer_mu);
  for (int d : devs) {
    for (int p : devs) {
      if (p == d) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, d, p) != cudaSuccess || !can) continue;
      cudaSetDevice(d);
      const cudaError_t e = cudaDeviceEnablePeerAccess(p, 0);
      if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) g_peer_on.insert({d, p});
      if (e != cudaSuccess) cudaGetLastError();
    }
  }
  cudaSetDevice(cur);
}
}  // namespace

bool peer_reachable(int from, int to) {
  if (from == to) return true;
  std::lock_guard<std::mutex> lock(g_peer_mu);
  return g_peer_on.count({from, to}) != 0;
}

void Runtime::init(const std::vector<int>& devices) {
  std::lock_guard<std::mutex> lock(mu_);
  std::vector<int> want = devices;
  if (want.empty()) {
    int count = 0;
    GPCX_CUDA(cudaGetDeviceCount(&count));
    for (int i = 0; i < count; ++i) want.push_back(i);
  }
  if (want.empty()) fail(Errc::TaskFailed, "no CUDA device available");
  std::vector<int> have;
  for (const Pool& p : pools_) have.push_back(p.device);
  if (inited_ && have == want) {
    // same set: quarantined devices are admitted again (if the context is
    // still broken, its next sticky error quarantines it again)
    for (Pool& p : pools_) {
      p.healthy = true;
      p.why.clear();
    }
    return;
  }
  pools_.clear();
  for (int d : want) {
    int count = 0;
    GPCX_CUDA(cudaGetDeviceCount(&count));
    if (d < 0 || d >= count) fail(Errc::BadValue, "device " + std::to_string(d) + " not present");
    pools_.push_back(Pool{d, {}, {}, true, {}});
  }
  enable_peer_access(want);
  inited_ = true;
}

void Runtime::shutdown() {
  std::lock_guard<std::mutex> lock(mu_);
  pools_.clear();
  inited_ = false;
}

void Runtime::ensure_init_locked() {
  if (inited_) return;
  int count = 0;
  GPCX_CUDA(cudaGetDeviceCount(&count));
  if (count <= 0) fail(Errc::TaskFailed, "no CUDA device available");
  std::vector<int> all;
  for (int i = 0; i < count; ++i) {
    pools_.push_back(Pool{i, {}, {}, true, {}});
    all.push_back(i);
  }
  enable_peer_access(all);
  inited_ = true;
}

std::vector<int> Runtime::devices() {
  std::lock_guard<std::mutex> lock(mu_);
  ensure_init_locked();
  std::vector<int> out;
  for (const Pool& p : pools_) out.push_back(p.device);
  return out;
}

int Runtime::device_at(int index) { return devices().at(static_cast<std::size_t>(index)); }

int Runtime::ndev() { return static_cast<int>(devices().size()); }

int Runtime::pick_device_index() {
  std::lock_guard<std::mutex> lock(mu_);
  ensure_init_locked();
  const int n = static_cast<int>(pools_.size());
  if (t_affinity >= 0 && t_affinity < n && pools_[t_affinity].healthy) return t_affinity;
  // round robin over the healthy devices
  for (int tries = 0; tries < n; ++tries) {
    const int i = static_cast<int>(rr_.fetch_add(1) % static_cast<unsigned>(n));
    if (pools_[i].healthy) return i;
  }
  std::string why = "no healthy device:";
  for (const Pool& p : pools_) why += " device " + std::to_string(p.device) + " quarantined (" + p.why + ");";
  fail(Errc::TaskFailed, why);
}

std::vector<int> Runtime::healthy_indices() {
  std::lock_guard<std::mutex> lock(mu_);
  ensure_init_locked();
  std::vector<int> out;
  for (std::size_t i = 0; i < pools_.size(); ++i)
    if (pools_[i].healthy) out.push_back(static_cast<int>(i));
  return out;
}

bool Runtime::healthy(int index) {
  std::lock_guard<std::mutex> lock(mu_);
  ensure_init_locked();
  return pools_.at(static_cast<std::size_t>(index)).healthy;
}

std::string Runtime::health_reason(int index) {
  std::lock_guard<std::mutex> lock(mu_);
  ensure_init_locked();
  return pools_.at(static_cast<std::size_t>(index)).why;
}

// Idle slots of a quarantined device are destroyed (their CUDA frees fail
// quietly on the dead context; the host-side objects go).
void Runtime::retire_idle_locked(Pool& pool) {
  for (Slot* s : pool.free) {
    for (std::size_t k = 0; k < pool.all.size(); ++k) {
      if (pool.all[k].get() == s) {
        pool.all.erase(pool.all.begin() + static_cast<std::ptrdiff_t>(k));
        break;
      }
    }
  }
  pool.free.clear();
  cudaGetLastError();
}

void Runtime::quarantine_device(int ordinal, const std::string& why) {
  std::lock_guard<std::mutex> lock(mu_);
  for (Pool& p : pools_) {
    if (p.device != ordinal || !p.healthy) continue;
    p.healthy = false;
    p.why = why;
    retire_idle_locked(p);
    std::fprintf(stderr, "gpcx: device %d quarantined after %s\n", ordinal, why.c_str());
  }
}

void Runtime::quarantine_index(int index, const std::string& why) {
  std::lock_guard<std::mutex> lock(mu_);
  ensure_init_locked();
  Pool& p = pools_.at(static_cast<std::size_t>(index));
  if (!p.healthy) return;
  p.healthy = false;
  p.why = why;
  retire_idle_locked(p);
}

SlotLease Runtime::acquire(int device_index) {
  std::unique_lock<std::mutex> lock(mu_);
  ensure_init_locked();
  Pool& pool = pools_.at(static_cast<std::size_t>(device_index));
  if (!pool.healthy)
    fail(Errc::TaskFailed, "device " + std::to_string(pool.device) + " quarantined (" + pool.why + ")");
  if (!pool.free.empty()) {
    Slot* s = pool.free.back();
    pool.free.pop_back();
    lock.unlock();
    use_device(s->device);
    return SlotLease(this, s);
  }
  const int device = pool.device;
  lock.unlock();
  auto slot = std::make_unique<Slot>();
  slot->device = device;
  use_device(device);
  GPCX_CUDA(cudaStreamCreateWithFlags(&slot->stream, cudaStreamNonBlocking));
  for (cudaEvent_t& e : slot->chunk_done)
    GPCX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  GPCX_CUDA(cudaEventCreateWithFlags(&slot->ready, cudaEventDisableTiming));
  slot->small.ensure(131072 + 256 + 65536 * 4 + sizeof(lut::PeerTable));
  slot->h_small.ensure(256);
  slot->lut_ws.ensure(lut::workspace_bytes(), /*zero=*/true);
  Slot* raw = slot.get();
  lock.lock();
  pool.all.push_back(std::move(slot));
  return SlotLease(this, raw);
}

void Runtime::release(Slot* slot) {
  std::lock_guard<std::mutex> lock(mu_);
  for (Pool& p : pools_) {
    if (p.device != slot->device) continue;
    for (std::size_t k = 0; k < p.all.size(); ++k) {
      if (p.all[k].get() != slot) continue;
      if (p.healthy) p.free.push_back(slot);
      else p.all.erase(p.all.begin() + static_cast<std::ptrdiff_t>(k));  // retired
      return;
    }
  }
  // Pool was rebuilt while the slot was leased: the unique_ptr that owned it
  // is gone already only if shutdown raced a request, which the C ABI
  // documents as unsupported; nothing to return it to.
}

namespace {
struct PinnedPool {
  std::mutex mu;
  std::vector<std::pair<std::uint64_t, void*>> idle;  // (capacity, ptr)
  std::uint64_t idle_bytes = 0;
};
PinnedPool& pinned_pool() {
  static PinnedPool* p = new PinnedPool();
  return *p;
}
std::atomic<std::uint64_t> g_pinned_in_use{0};
// Page-locked bytes leased at once (GPCX_PINNED_CAP_MB, default 32 GiB).
// Idle pooled buffers are kept up to the same bound: freeing and
// re-registering page-locked memory costs ~ms per GiB (cudaFreeHost /
// cudaHostAlloc serialise with the whole context), so a server whose
// in-flight staging exceeds a smaller idle cap churns on every request.
std::uint64_t pinned_cap() {
  static const std::uint64_t cap = [] {
    const char* v = std::getenv("GPCX_PINNED_CAP_MB");
    const long long mb = v != nullptr ? std::atoll(v) : 0;
    return mb > 0 ? static_cast<std::uint64_t>(mb) << 20 : 32ull << 30;
  }();
  return cap;
}
}  // namespace

std::uint64_t pinned_in_use() { return g_pinned_in_use.load(); }

PinnedLease& PinnedLease::operator=(PinnedLease&& o) noexcept {
  if (this != &o) {
    this->~PinnedLease();
    ptr_ = o.ptr_;
    cap_ = o.cap_;
    pageable_ = o.pageable_;
    o.ptr_ = nullptr;
  }
  return *this;
}

PinnedLease::~PinnedLease() {
  if (ptr_ == nullptr) return;
  if (pageable_) {
    std::free(ptr_);
    ptr_ = nullptr;
    return;
  }
  g_pinned_in_use.fetch_sub(cap_);
  PinnedPool& pool = pinned_pool();
  std::lock_guard<std::mutex> lock(pool.mu);
  if (pool.idle_bytes + cap_ > pinned_cap()) {
    cudaFreeHost(ptr_);
  } else {
    pool.idle.emplace_back(cap_, ptr_);
    pool.idle_bytes += cap_;
  }
  ptr_ = nullptr;
}

PinnedLease pinned_acquire(std::uint64_t bytes) {
  std::uint64_t cls = 4096;
  while (cls < bytes) cls <<= 1;
  // over the page-locked budget: a heap lease (staged through the slots'
  // pinned bounce buffers by h2d / d2h)
  if (g_pinned_in_use.fetch_add(cls) + cls > pinned_cap()) {
    g_pinned_in_use.fetch_sub(cls);
    void* p = std::malloc(cls);
    if (p == nullptr) fail(Errc::TaskFailed, "out of host memory");
    return PinnedLease(p, cls, /*pageable=*/true);
  }
  PinnedPool& pool = pinned_pool();
  {
    std::lock_guard<std::mutex> lock(pool.mu);
    for (std::size_t i = 0; i < pool.idle.size(); ++i) {
      if (pool.idle[i].first == cls) {
        void* p = pool.idle[i].second;
        pool.idle.erase(pool.idle.begin() + static_cast<std::ptrdiff_t>(i));
        pool.idle_bytes -= cls;
        return PinnedLease(p, cls);
      }
    }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, cls, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    g_pinned_in_use.fetch_sub(cls);
    p = std::malloc(cls);
    if (p == nullptr) fail(Errc::TaskFailed, "out of host memory");
    return PinnedLease(p, cls, /*pageable=*/true);
  }
  return PinnedLease(p, cls);
}

void pinned_trim() {
  PinnedPool& pool = pinned_pool();
  std::lock_guard<std::mutex> lock(pool.mu);
  for (auto& e : pool.idle) cudaFreeHost(e.second);
  pool.idle.clear();
  pool.idle_bytes = 0;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

namespace {
struct ArrivalRegistry {
  std::mutex mu;
  std::vector<Arrival*> live;
};
ArrivalRegistry& arrivals() {
  static ArrivalRegistry* r = new ArrivalRegistry();
  return *r;
}
Arrival* find_arrival(const void* p) {
  ArrivalRegistry& r = arrivals();
  std::lock_guard<std::mutex> lock(r.mu);
  const auto* b = static_cast<const std::uint8_t*>(p);
  for (Arrival* a : r.live)
    if (b >= a->base() && b < a->base() + a->size()) return a;
  return nullptr;
}
}  // namespace

Arrival::Arrival(const void* base, std::uint64_t len)
    : base_(static_cast<const std::uint8_t*>(base)), len_(len) {
  ArrivalRegistry& r = arrivals();
  std::lock_guard<std::mutex> lock(r.mu);
  r.live.push_back(this);
}

Arrival::~Arrival() {
  ArrivalRegistry& r = arrivals();
  std::lock_guard<std::mutex> lock(r.mu);
  for (std::size_t i = 0; i < r.live.size(); ++i) {
    if (r.live[i] == this) {
      r.live.erase(r.live.begin() + static_cast<std::ptrdiff_t>(i));
      break;
    }
  }
}

void Arrival::advance(std::uint64_t got) {
  {
    std::lock_guard<std::mutex> lock(mu_);
    got_ = got;
  }
  cv_.notify_all();
}

void Arrival::fail() {
  {
    std::lock_guard<std::mutex> lock(mu_);
    failed_ = true;
  }
  cv_.notify_all();
}

void Arrival::wait_for(std::uint64_t upto) {
  std::unique_lock<std::mutex> lock(mu_);
  cv_.wait(lock, [&] { return failed_ || got_ >= upto; });
  if (got_ < upto) gpcx::fail(Errc::Truncated, "request payload ended early");
}

void h2d(Slot& s, void* dst, const void* src, std::uint64_t bytes) {
  if (bytes == 0) return;
  const obs::Range range("h2d");
  if (Arrival* a = find_arrival(src)) {  // payload still arriving: chunk as it lands
    const std::uint64_t start = static_cast<std::uint64_t>(static_cast<const std::uint8_t*>(src) - a->base());
    const auto* in = static_cast<const std::uint8_t*>(src);
    auto* out = static_cast<std::uint8_t*>(dst);
    for (std::uint64_t off = 0; off < bytes; off += kArrivalChunk) {
      const std::uint64_t len = std::min(kArrivalChunk, bytes - off);
      a->wait_for(start + off + len);
      GPCX_CUDA(cudaMemcpyAsync(out + off, in + off, len, cudaMemcpyHostToDevice, s.stream));
    }
    return;
  }
  if (is_pinned(src)) {
    GPCX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s.stream));
    return;
  }
  const std::uint64_t chunk = std::min<std::uint64_t>(kStageChunk, bytes);
  s.stage[0].ensure(chunk);
  s.stage[1].ensure(chunk);
  const auto* in = static_cast<const unsigned char*>(src);
  auto* out = static_cast<unsigned char*>(dst);
  std::uint64_t off = 0;
  for (int i = 0; off < bytes; ++i, off += chunk) {
    const std::uint64_t len = std::min(chunk, bytes - off);
    PinnedBuf& st = s.stage[i & 1];
    GPCX_CUDA(cudaEventSynchronize(s.chunk_done[i & 1]));  // previous DMA out of st
    std::memcpy(st.ptr, in + off, len);
    GPCX_CUDA(cudaMemcpyAsync(out + off, st.ptr, len, cudaMemcpyHostToDevice, s.stream));
    GPCX_CUDA(cudaEventRecord(s.chunk_done[i & 1], s.stream));
  }
}

void d2h(Slot& s, void* dst, const void* src, std::uint64_t bytes) {
  const obs::Range range("d2h");
  if (bytes == 0) {
    GPCX_CUDA(cudaStreamSynchronize(s.stream));
    return;
  }
  if (is_pinned(dst)) {
    GPCX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s.stream));
    GPCX_CUDA(cudaStreamSynchronize(s.stream));
    return;
  }
  const std::uint64_t chunk = std::min<std::uint64_t>(kStageChunk, bytes);
  s.stage[0].ensure(chunk);
  s.stage[1].ensure(chunk);
  const auto* in = static_cast<const unsigned char*>(src);
  auto* out = static_cast<unsigned char*>(dst);
  const std::uint64_t nchunks = (bytes + chunk - 1) / chunk;
  auto issue = [&](std::uint64_t i) {
    const std::uint64_t off = i * chunk;
    const std::uint64_t len = std::min(chunk, bytes - off);
    GPCX_CUDA(cudaMemcpyAsync(s.stage[i & 1].ptr, in + off, len, cudaMemcpyDeviceToHost,
                              s.stream));
    GPCX_CUDA(cudaEventRecord(s.chunk_done[i & 1], s.stream));
  };
  issue(0);
  for (std::uint64_t i = 0; i < nchunks; ++i) {
    if (i + 1 < nchunks) issue(i + 1);
    GPCX_CUDA(cudaEventSynchronize(s.chunk_done[i & 1]));
    const std::uint64_t off = i * chunk;
    std::memcpy(out + off, s.stage[i & 1].ptr, std::min(chunk, bytes - off));
  }
}

}  // namespace gpcx::rt
