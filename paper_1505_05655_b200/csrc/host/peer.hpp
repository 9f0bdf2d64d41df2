// peer.hpp -- one rank of a multi-GPU LUT group whose histogram exchange
// runs inside the fused kernel over peer memory (kernels.hpp: PeerTable).
//
// LUT_GEN / LUT_CORRECT shard into row bands with ONE
// exchange step, the 65536-bin histogram sum.  With one process per GPU
// (bench.py under torchrun) every rank owns a device block
//   [hist parity 0 | hist parity 1 | flag rows | PeerTable]
// allocated with cudaMalloc, exports it as a CUDA IPC handle, and maps the
// peers' blocks (cudaIpcOpenMemHandle: an NVLink P2P mapping between GPUs,
// or a plain second mapping on one GPU).  Each call is then ONE cooperative
// launch per rank -- count, publish + rendezvous, sum of the peers'
// slices, LUT, apply -- instead of count, NCCL all-reduce, build + apply.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../kernels.hpp"

namespace gpcx::peer {

using lut::kMaxRanks;
using lut::kPeerBlockBytes;
using lut::kPeerFlagBytes;
using lut::kPeerHistBytes;
using lut::PeerTable;

class LutRank {
 public:
  LutRank(int rank, int nranks);  // on the current device
  ~LutRank();
  LutRank(const LutRank&) = delete;
  LutRank& operator=(const LutRank&) = delete;

  cudaIpcMemHandle_t handle() const;
  // handles[r] for r in [0, nranks): opens every peer's block (own entry
  // ignored) and uploads the rank's PeerTable.
  void connect(const cudaIpcMemHandle_t* handles);

  // One step of the group: every rank must make the same sequence of
  // calls (each call advances the shared sequence number).
  void correct(const std::uint16_t* in, std::uint16_t* out, std::uint64_t n, int mode,
               std::uint16_t* lut, gpcx_lut_stats* stats, void* ws, cudaStream_t stream,
               std::uint64_t ws_bytes = 0);

  int rank() const { return rank_; }
  int nranks() const { return nranks_; }

 private:
  std::uint32_t* hist_at(unsigned char* block, int parity) const;
  int device_ = 0, rank_ = 0, nranks_ = 1;
  unsigned char* block_ = nullptr;
  std::vector<unsigned char*> opened_;
  PeerTable* d_table_ = nullptr;
  bool connected_ = false;
  std::uint32_t seq_ = 0;
  std::uint64_t timeout_ns_ = 0;
};

}  // namespace gpcx::peer
