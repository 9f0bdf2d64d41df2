// runtime.cpp -- see runtime.hpp.
#include "runtime.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>

#include "../cuda_util.hpp"
#include "../kernels.hpp"

namespace gpcx::rt {

void use_device(int device) { GPCX_CUDA(cudaSetDevice(device)); }

void DeviceBuf::ensure(std::uint64_t bytes, bool zero) {
  if (bytes <= cap && ptr != nullptr) return;
  release();
  const std::uint64_t want = std::max<std::uint64_t>(bytes, 256);
  GPCX_CUDA(cudaMalloc(&ptr, want));
  cap = want;
  if (zero) GPCX_CUDA(cudaMemset(ptr, 0, want));
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
  if (inited_ && have == want) return;
  pools_.clear();
  for (int d : want) {
    int count = 0;
    GPCX_CUDA(cudaGetDeviceCount(&count));
    if (d < 0 || d >= count) fail(Errc::BadValue, "device " + std::to_string(d) + " not present");
    pools_.push_back(Pool{d, {}, {}});
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
    pools_.push_back(Pool{i, {}, {}});
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
  const int n = ndev();
  return static_cast<int>(rr_.fetch_add(1) % static_cast<unsigned>(n));
}

SlotLease Runtime::acquire(int device_index) {
  std::unique_lock<std::mutex> lock(mu_);
  ensure_init_locked();
  Pool& pool = pools_.at(static_cast<std::size_t>(device_index));
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
    for (auto& owned : p.all) {
      if (owned.get() == slot) {
        p.free.push_back(slot);
        return;
      }
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
constexpr std::uint64_t kPinnedIdleCap = 8ull << 30;
}  // namespace

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
  PinnedPool& pool = pinned_pool();
  std::lock_guard<std::mutex> lock(pool.mu);
  if (pool.idle_bytes + cap_ > kPinnedIdleCap) {
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
