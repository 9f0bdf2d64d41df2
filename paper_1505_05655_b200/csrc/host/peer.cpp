// peer.cpp -- see peer.hpp.
#include "peer.hpp"

#include <cstdlib>
#include <string>

#include "../cuda_util.hpp"

namespace gpcx::peer {

namespace {
std::uint64_t timeout_from_env() {
  // GPCX_PEER_TIMEOUT_MS: how long a rank waits for its peers inside the
  // kernel before trapping (a dead peer must not hang the GPU)
  const char* v = std::getenv("GPCX_PEER_TIMEOUT_MS");
  const long long ms = v != nullptr ? std::atoll(v) : 60000;
  return static_cast<std::uint64_t>(ms > 0 ? ms : 60000) * 1000000ull;
}
}  // namespace

LutRank::LutRank(int rank, int nranks) : rank_(rank), nranks_(nranks) {
  if (nranks < 1 || nranks > kMaxRanks)
    fail(Errc::BadValue, "peer group of " + std::to_string(nranks) + " ranks (1.." +
                             std::to_string(kMaxRanks) + ")");
  if (rank < 0 || rank >= nranks)
    fail(Errc::BadValue, "rank " + std::to_string(rank) + " of " + std::to_string(nranks));
  GPCX_CUDA(cudaGetDevice(&device_));
  GPCX_CUDA(cudaMalloc(&block_, kPeerBlockBytes));
  // flags start at 0 and the first call uses seq 1
  GPCX_CUDA(cudaMemset(block_, 0, kPeerBlockBytes));
  GPCX_CUDA(cudaDeviceSynchronize());
  d_table_ = reinterpret_cast<PeerTable*>(block_ + kPeerHistBytes + kPeerFlagBytes);
  timeout_ns_ = timeout_from_env();
}

LutRank::~LutRank() {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device_);
  cudaDeviceSynchronize();
  for (unsigned char* p : opened_) cudaIpcCloseMemHandle(p);
  if (block_ != nullptr) cudaFree(block_);
  cudaSetDevice(cur);
}

cudaIpcMemHandle_t LutRank::handle() const {
  cudaIpcMemHandle_t h;
  GPCX_CUDA(cudaIpcGetMemHandle(&h, block_));
  return h;
}

std::uint32_t* LutRank::hist_at(unsigned char* block, int parity) const {
  return reinterpret_cast<std::uint32_t*>(block + parity * (kPeerHistBytes / 2));
}

void LutRank::connect(const cudaIpcMemHandle_t* handles) {
  if (connected_) fail(Errc::BadValue, "peer group already connected");
  GPCX_CUDA(cudaSetDevice(device_));
  PeerTable t;
  t.rank = rank_;
  t.nranks = nranks_;
  for (int r = 0; r < nranks_; ++r) {
    unsigned char* base = block_;
    if (r != rank_) {
      void* p = nullptr;
      GPCX_CUDA(cudaIpcOpenMemHandle(&p, handles[r], cudaIpcMemLazyEnablePeerAccess));
      base = static_cast<unsigned char*>(p);
      opened_.push_back(base);
    }
    t.flags[r] = reinterpret_cast<std::uint32_t*>(base + kPeerHistBytes);
    t.hist[0][r] = hist_at(base, 0);
    t.hist[1][r] = hist_at(base, 1);
  }
  GPCX_CUDA(cudaMemcpy(d_table_, &t, sizeof(t), cudaMemcpyHostToDevice));
  connected_ = true;
}

void LutRank::correct(const std::uint16_t* in, std::uint16_t* out, std::uint64_t n, int mode,
                      std::uint16_t* lut, gpcx_lut_stats* stats, void* ws,
                      cudaStream_t stream, std::uint64_t ws_bytes) {
  if (!connected_) fail(Errc::BadValue, "peer group not connected");
  GPCX_CUDA(cudaSetDevice(device_));
  const std::uint32_t seq = ++seq_;
  lut::launch_correct_peer(d_table_, hist_at(block_, seq & 1), seq, timeout_ns_, in, out, n,
                           mode, lut, stats, ws, stream, ws_bytes);
}

}  // namespace gpcx::peer
