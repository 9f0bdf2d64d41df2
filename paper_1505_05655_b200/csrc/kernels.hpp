// kernels.hpp -- host-side launchers of the sm_100a kernels.
//
// All launchers are asynchronous on the given stream and throw
// gpcx::Error(TaskFailed) on a launch failure.  Shapes are validated by the
// callers (capi.cpp); launchers assume valid arguments.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/gpcx.h"

namespace gpcx {

namespace lut {

inline constexpr int kBins = 65536;
inline constexpr int kWords = kBins / 2;      // u16 pairs per u32 word
inline constexpr int kMaxParts = 296;         // per-CTA partial histograms

// Workspace layout (bytes):
//   [0, 256 Ki)               overflow counters, u32[65536] (self-cleaning)
//   [256 Ki, 512 Ki)          merged histogram, u32[65536]
//   [512 Ki, +kMaxParts*8)    per-CTA (lo, hi) pairs for the min/max path
//   [.. , + kMaxParts*128 Ki) per-CTA packed partial histograms
//   [workspace_bytes(), +plane_bytes(n))  the residual plane of an n-sample
//                             LUT_CORRECT (lut.cu); absent below 2^25 samples
std::uint64_t workspace_bytes();
// Recommended size for n samples (fixed part + residual plane).  Launchers
// given a workspace of at least this size code the plane; one of at least
// workspace_bytes() is enough for every path.
std::uint64_t workspace_bytes(std::uint64_t n);
std::uint64_t plane_bytes(std::uint64_t n);
// The merged-histogram scratch inside a workspace (u32[65536]).
std::uint32_t* ws_hist(void* ws);

int parts_for(std::uint64_t n, int num_sms);

// ---- multi-GPU histogram exchange over peer memory (no NCCL) ----------
// Rank r of a group publishes its band histogram in its own HBM; the fused
// kernel of every rank sums the group's histograms slice by slice with
// system-scope loads of the peers' buffers (NVLink P2P / CUDA IPC
// mappings).  Two ways to order it:
//   flags != nullptr  device-side: after writing slice b, rank r's slice
//                     CTA b stores seq into flags[q][b][r] of every rank q
//                     (release, system scope) and waits until its own
//                     flags[r][b][*] >= seq (acquire) -- one launch per step
//                     and no host round trip (one process per GPU);
//   flags == nullptr  host-ordered: the caller guarantees every rank's
//                     histogram is complete before the launch (the
//                     in-process planner joins its band threads).
// Histogram buffers are double-buffered by seq parity, so a rank that runs
// ahead into step seq+1 never overwrites what a slower peer still reads.
inline constexpr int kMaxRanks = 8;
inline constexpr int kFlagSlices = 128;  // one flag row per phase-2 slice CTA
struct PeerTable {
  int rank = 0, nranks = 1;
  std::uint32_t* flags[kMaxRanks] = {};    // rank q's flag block: [kFlagSlices][kMaxRanks] u32
  std::uint32_t* hist[2][kMaxRanks] = {};  // rank q's histogram (u32[65536]) by seq parity
};
// One rank's device block: hist[2][65536] u32 | flags | its PeerTable.
inline constexpr std::uint64_t kPeerHistBytes = 2ull * kBins * 4;
inline constexpr std::uint64_t kPeerFlagBytes = std::uint64_t(kFlagSlices) * kMaxRanks * 4;
inline constexpr std::uint64_t kPeerBlockBytes = kPeerHistBytes + kPeerFlagBytes + 4096;
// LUT_CORRECT / LUT_GEN of one rank's band with the exchange fused into the
// cooperative kernel: stages count (+ publish) -> exchange -> LUT -> apply
// (out == nullptr: LUT only).  `table` is the device copy of the rank's
// PeerTable, `own_hist` = its hist[seq & 1][rank].
void launch_correct_peer(const PeerTable* table, std::uint32_t* own_hist, std::uint32_t seq,
                         std::uint64_t timeout_ns, const std::uint16_t* in, std::uint16_t* out,
                         std::uint64_t n, int mode, std::uint16_t* lut, gpcx_lut_stats* stats,
                         void* ws, cudaStream_t stream, std::uint64_t ws_bytes = 0);
// Host-ordered second half for the in-process planner: sum the group's
// published histograms (table->flags unused), LUT, apply the band.
// ws_bytes (optional): the band's count launch (launch_hist with the same
// ws_bytes, same image and workspace) coded the residual plane, read here.
void launch_correct_from_peers(const PeerTable* table, std::uint32_t seq, int mode,
                               const std::uint16_t* in, std::uint16_t* out, std::uint64_t n,
                               std::uint16_t* lut, gpcx_lut_stats* stats, void* ws,
                               cudaStream_t stream, std::uint64_t ws_bytes = 0);

// Histogram of img into hist (u32[65536]).  ws_bytes >= workspace_bytes(n)
// also codes the residual plane for a later launch_correct_from_peers of the
// same image and workspace (the in-process planner); 0 never does.
void launch_hist(const std::uint16_t* img, std::uint64_t n, std::uint32_t* hist,
                 void* ws, cudaStream_t stream, std::uint64_t ws_bytes = 0);
// LUT + stats from a merged histogram (`ws` is a LUT workspace, used for the
// per-slice scan summaries).
void launch_from_hist(const std::uint32_t* hist, int mode, std::uint16_t* lut,
                      gpcx_lut_stats* stats, void* ws, cudaStream_t stream);
// LUT from a merged (e.g. all-reduced) histogram, then out = LUT[in]: one
// launch when in/out are co-aligned.  The second half of a sharded LUT_CORRECT.
void launch_correct_from_hist(const std::uint32_t* hist, int mode, const std::uint16_t* in,
                              std::uint16_t* out, std::uint64_t n, std::uint16_t* lut,
                              gpcx_lut_stats* stats, void* ws, cudaStream_t stream);
// Single-device LUT_GEN equalize: one cooperative fused_kernel launch
// (the histogram lands in ws_hist(ws)).
void launch_hist_lut(const std::uint16_t* img, std::uint64_t n, int mode, std::uint16_t* lut,
                     gpcx_lut_stats* stats, void* ws, cudaStream_t stream);
// Single-device LUT_CORRECT (LUT_GEN + apply; in == out allowed): equalize
// with co-aligned buffers is ONE fused_kernel launch; otherwise gen + apply.
void launch_correct(const std::uint16_t* in, std::uint16_t* out, std::uint64_t n, int mode,
                    std::uint16_t* lut, gpcx_lut_stats* stats, void* ws, cudaStream_t stream,
                    std::uint64_t ws_bytes = 0);
void launch_minmax(const std::uint16_t* img, std::uint64_t n,
                   gpcx_lut_stats* stats, void* ws, cudaStream_t stream);
void launch_from_minmax(const gpcx_lut_stats* stats, std::uint16_t* lut,
                        cudaStream_t stream);
void launch_apply(const std::uint16_t* lut, const std::uint16_t* in,
                  std::uint16_t* out, std::uint64_t n, cudaStream_t stream);

}  // namespace lut

namespace demosaic {
// BAYER_BILINEAR (gradient=false) / BAYER_GRADIENT on a rows x cols u16
// mosaic -> 3 planes (R || G || B); phase = gpc::img::CfaPhase ordinal
// (RGGB, BGGR, GRBG, GBRG).  BadImage below 2x2 like BayerImage::validate.
void launch(bool gradient, int phase, const std::uint16_t* in, std::uint16_t* out,
            std::uint64_t rows, std::uint64_t cols, cudaStream_t stream);
// Output rows [row_base, row_base + out_rows) into three band-local planes
// (out_rows x cols each); `in` holds image rows from in_row0 on, which must
// include the band's halo rows (in_row0 <= max(row_base - 1, 0)).
void launch_band(bool gradient, int phase, const std::uint16_t* in, std::uint16_t* out,
                 std::uint64_t rows, std::uint64_t cols, std::uint64_t row_base,
                 std::uint64_t in_row0, std::uint64_t out_rows, cudaStream_t stream);
}  // namespace demosaic

namespace lsq {
inline constexpr int kMaxOrder = 8;  // gpc::lsq::kMaxOrder
// Per-line polynomial fits of `lines` x `pixels` samples (f32 or f64,
// device memory).  out_coeffs: lines x (kMaxOrder + 2) doubles, the first
// order+1 the coefficients (constant first) then the SSE; out_status:
// lines x 4 doubles {code (0 ok, 1 non-finite, 2 insufficient points,
// 3 singular), col / index, best pivot, pivot floor}.
std::uint64_t workspace_bytes(std::uint64_t lines, std::uint64_t pixels);
void launch(const void* y, bool dtype_f32, std::uint64_t lines, std::uint64_t pixels, int order,
            double* out_coeffs, double* out_status, void* ws, cudaStream_t stream);
}  // namespace lsq

namespace synth {
void launch_image(int kind, std::uint64_t seed, std::uint64_t rows,
                  std::uint64_t cols, std::uint64_t row0, std::uint64_t nrows,
                  std::uint16_t* out, cudaStream_t stream);
void launch_matrix(int kind, std::uint64_t seed, std::uint64_t rows,
                   std::uint64_t cols, std::uint64_t row0, std::uint64_t nrows,
                   float* out, cudaStream_t stream);
void launch_digest(const std::uint16_t* v, std::uint64_t n,
                   std::uint64_t index0, std::uint64_t* digest,
                   cudaStream_t stream);
// out[j] = c[rc[j].row * ldc + rc[j].col] for `count` (u32 row, u32 col)
// pairs in device memory (sampled entries of a synthetic MATMUL).
void launch_gather(const float* c, std::uint64_t ldc, const void* rc, std::uint32_t count,
                   float* out, cudaStream_t stream);
// The generators' hash, on the host (seeds, sample positions).
std::uint64_t splitmix64_host(std::uint64_t x);
// A kernel that executes __trap() (gpcx_debug_fault: a real sticky error).
void launch_trap(cudaStream_t stream);
}  // namespace synth

namespace gemm {
// SIMT FP32 (reference precision).  The workspace (sgemm_workspace_bytes:
// A^T for aligned shapes, else 0) selects the fastest kernel; without it
// the same bits come from the row-major-A kernel.
std::uint64_t sgemm_workspace_bytes(std::uint64_t m, std::uint64_t n, std::uint64_t k);
void launch_sgemm(std::uint64_t m, std::uint64_t n, std::uint64_t k,
                  const float* A, std::uint64_t lda, const float* B,
                  std::uint64_t ldb, float* C, std::uint64_t ldc,
                  void* ws, std::uint64_t ws_bytes, cudaStream_t stream);
// Tensor-core path (tcgen05): prec = GPCX_PREC_TF32 / GPCX_PREC_BF16.
std::uint64_t tc_workspace_bytes(int prec, std::uint64_t m, std::uint64_t n,
                                 std::uint64_t k);
void launch_tc(int prec, std::uint64_t m, std::uint64_t n, std::uint64_t k,
               const float* A, std::uint64_t lda, const float* B,
               std::uint64_t ldb, float* C, std::uint64_t ldc, void* ws,
               cudaStream_t stream);
}  // namespace gemm

int device_sm_count();  // SMs of the current device (cached per device)

}  // namespace gpcx
