// tc_gemm.cu -- tensor-core MATMUL (prec = bf16 | tf32) for sm_100a:
// TMA-fed, mbarrier-pipelined, warp-specialised tcgen05 GEMM with the
// accumulators in TMEM.
//
// Contract: SURVEY.md §8a' a'4 -- C (m x n, f32 row-major) = A (m x k) x
// B (k x n), f32 row-major inputs.  The tensor path rounds the operands
// once (bf16: RNE, tf32: RNA -- exactly what oracle/gpcx_oracle.c's
// orc_round_matrix does), accumulates in fp32 in TMEM and writes f32.
//
// Pipeline per call:
//   prep_a_kernel   A f32 -> A' (m x Kp, K-major, bf16 or tf32-in-f32)
//   prep_bt_kernel  B f32 -> B'^T (n x Kp, K-major): smem-tiled transpose
//   gemm_kernel     persistent, one CTA per SM, 128 x 256 output tile,
//                   4-stage TMA ring (128B swizzle), 64 bf16 / 32 tf32 of K
//                   per stage; warp 0 = TMA producer, warp 1 = MMA issuer
//                   (one thread issues tcgen05.mma 128x256xK16/K8), warp 2
//                   = TMEM allocator, warps 4-7 = epilogue (tcgen05.ld
//                   32x32b -> registers -> global).  The 2 x 256 TMEM
//                   accumulator columns are double-buffered so tile i's
//                   epilogue overlaps tile i+1's MMAs.
// Kp = k rounded up to the K tile; the zero padding makes every K tile
// whole, and TMA zero-fills rows past m / n.  The K order per output is
// fixed (tile by tile, ascending), so C is bitwise identical for any
// block-row sharding across GPUs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>

#include "cuda_util.hpp"
#include "kernels.hpp"

namespace gpcx::gemm {

namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int kStages = 4;
constexpr int kStageBytesA = BM * 128;  // 128 bytes of K per row
constexpr int kStageBytesB = BN * 128;
constexpr int kStageBytes = kStageBytesA + kStageBytesB;
constexpr int kThreads = 256;           // 8 warps
constexpr int kEpiWarp0 = 4;
constexpr int kTmemCols = 512;          // 2 accumulator buffers x 256 columns
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

// ------------------------------------------------------------------ PTX ---

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ std::uint64_t global_ns() {
  std::uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Parity wait with a watchdog: a pipeline bug traps after ~10 s (a launch
// error the host reports as ERR:TASK_FAILED) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
  const std::uint32_t addr = smem_u32(bar);
  std::uint32_t done = 0;
  std::uint64_t t0 = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if (t0 == 0) t0 = global_ns();
    else if (global_ns() - t0 > 10000000000ull) __trap();
  }
}

// The epilogue's wait for an accumulator (~a tile's mainloop, 100s of us):
// back off with __nanosleep between probes so the four waiting warps do not
// spin (power-capped GEMM: idle issue slots are energy the clock can use).
__device__ __forceinline__ void mbar_wait_sleepy(std::uint64_t* bar, std::uint32_t parity) {
  const std::uint32_t addr = smem_u32(bar);
  std::uint32_t done = 0;
  std::uint64_t t0 = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
#ifndef GPCX_NO_SLEEPY
    __nanosleep(2000);
#endif
    if (t0 == 0) t0 = global_ns();
    else if (global_ns() - t0 > 10000000000ull) __trap();
  }
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, std::uint64_t* bar, void* dst,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

template <bool kTf32>
__device__ __forceinline__ void tc_mma(std::uint32_t tmem_d, std::uint64_t adesc,
                                       std::uint64_t bdesc, std::uint32_t idesc,
                                       std::uint32_t accumulate) {
  if constexpr (kTf32) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// K-major, 128-byte-swizzled operand tile: rows of 128 B, 8-row atoms of
// 1 KiB stacked at SBO = 1024 B; LBO unused for swizzled K-major (1).
__device__ __forceinline__ std::uint64_t smem_desc(const void* tile) {
  const std::uint64_t addr = smem_u32(tile);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | (static_cast<std::uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: f32 accumulate, A/B = bf16 (1) or tf32 (2), both
// K-major, N >> 3 at bit 17, M >> 4 at bit 24.
template <bool kTf32, int kM = BM, int kN = BN>
__host__ __device__ constexpr std::uint32_t instr_desc() {
  const std::uint32_t fmt = kTf32 ? 2u : 1u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<std::uint32_t>(kN >> 3) << 17) |
         (static_cast<std::uint32_t>(kM >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld32(std::uint32_t taddr, std::uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Tile raster: groups of `group_m` m-blocks swept n-block by n-block, so the
// tiles resident at once (one wave of persistent CTAs) cover a near-square
// block of C and read the fewest distinct A / B rows per K step -- the
// operand panels of a wave come from DRAM once and are L2 hits for every
// other CTA of the wave.  1-SM 128x256 tiles: 16 x ~9 blocks per wave;
// CTA-pair 256x256 tiles: 8 x ~9.
struct TileMap {
  int mt, nt, group_m;
  __device__ __forceinline__ void coords(int t, int& mb, int& nb) const {
    const int per_group = group_m * nt;
    const int g = t / per_group;
    const int first_m = g * group_m;
    const int gm = min(group_m, mt - first_m);
    const int r = t - g * per_group;
    mb = first_m + r % gm;
    nb = r / gm;
  }
};

template <bool kTf32>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                float* __restrict__ C, int m, int n, std::uint64_t ldc, int ktiles, int mt, int nt) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  // 1 KiB alignment for the 128B-swizzle atoms.
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~static_cast<std::uintptr_t>(1023));
  std::uint8_t* tiles = smem;
  auto* bars = reinterpret_cast<std::uint64_t*>(smem + kStages * kStageBytes);
  std::uint64_t* full = bars;                    // [kStages]
  std::uint64_t* empty = bars + kStages;         // [kStages]
  std::uint64_t* tmem_full = bars + 2 * kStages; // [2]
  std::uint64_t* tmem_empty = tmem_full + 2;     // [2]
  auto* tmem_slot = reinterpret_cast<std::uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TileMap tm{mt, nt, 16};
  const int ntiles = mt * nt;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      std::uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int mb, nb;
        tm.coords(t, mb, nb);
        for (int kb = 0; kb < ktiles; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          std::uint8_t* sa = tiles + stage * kStageBytes;
          mbar_expect_tx(&full[stage], kStageBytes);
          const int kx = kb * (kTf32 ? 32 : 64);
          tma_load_2d(&map_a, &full[stage], sa, kx, mb * BM);
          tma_load_2d(&map_b, &full[stage], sa + kStageBytesA, kx, nb * BN);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      constexpr std::uint32_t idesc = instr_desc<kTf32>();
      int stage = 0;
      std::uint32_t phase = 0;
      int acc = 0;
      std::uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const std::uint32_t tmem_d = tmem_base + static_cast<std::uint32_t>(acc * BN);
        for (int kb = 0; kb < ktiles; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const std::uint8_t* sa = tiles + stage * kStageBytes;
          const std::uint64_t adesc = smem_desc(sa);
          const std::uint64_t bdesc = smem_desc(sa + kStageBytesA);
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 4 x 32 bytes of K per 128-byte row
            tc_mma<kTf32>(tmem_d, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          tc_commit(&empty[stage]);  // frees the smem slot when these MMAs finish
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tmem_full[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ---------------- epilogue: TMEM -> registers -> C ----------------
    const int quarter = warp - kEpiWarp0;  // TMEM lanes 32*quarter ..
    int acc = 0;
    std::uint32_t acc_phase = 0;
    const bool vec_ok = (ldc % 4 == 0) && ((reinterpret_cast<std::uintptr_t>(C) & 15) == 0);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int mb, nb;
      tm.coords(t, mb, nb);
      mbar_wait_sleepy(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int row = mb * BM + quarter * 32 + lane;
      float* crow = C + static_cast<std::uint64_t>(row) * ldc;
      const std::uint32_t taddr =
          tmem_base + (static_cast<std::uint32_t>(quarter * 32) << 16) + static_cast<std::uint32_t>(acc * BN);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        std::uint32_t v[32];
        tmem_ld32(taddr + c, v);
        const int col = nb * BN + c;
        if (row < m) {
          if (vec_ok && col + 32 <= n) {
            float4* dst = reinterpret_cast<float4*>(crow + col);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                   __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < n) crow[col + j] = __uint_as_float(v[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// ------------------------------------------------- CTA-pair (2-SM) kernel ---
//
// Two CTAs of a cluster on a TPC form one 256 x 256 tile: CTA r holds rows
// [128r, 128r+128) of the A tile and rows [128r, 128r+128) of the B'^T tile
// (N half) at identical smem offsets; the leader (rank 0) issues
// tcgen05.mma.cta_group::2 M=256 N=256, which reads both CTAs' smem and
// writes both CTAs' TMEM (rows 0-127 in the leader, 128-255 in the peer).
// Per CTA a stage is 32 KiB (half of the 1-SM kernel's B), so the ring is
// 6 deep for the same smem, and each SM's tensor-core smem reads halve.
// Barrier protocol (as CUTLASS's 2SM pipeline): both producers wait on
// their own `empty` slot (the leader's commit multicasts to both CTAs),
// issue cta_group::2 TMA loads that complete_tx on the LEADER's `full`
// barrier, and only the leader arms it with the pair's total bytes.  The
// accumulator-ready commit multicasts to both CTAs' tmem_full; all 8
// epilogue warps of the pair arrive on the leader's tmem_empty.

constexpr int kStageBytes2 = 2 * 128 * 128;  // A half + B half, 16 KiB each
template <int S>
constexpr int smem_bytes2() {
  return S * kStageBytes2 + 1024 + 256;
}
constexpr std::uint32_t kPeerMask = 0xFEFFFFFFu;  // rank bit of a shared::cluster address

__device__ __forceinline__ std::uint32_t cta_rank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, std::uint32_t leader_bar,
                                                 void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}

__device__ __forceinline__ void tc_commit_pair(std::uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
          "r"(smem_u32(bar)),
      "h"(static_cast<std::uint16_t>(0x3))
      : "memory");
}

template <bool kTf32>
__device__ __forceinline__ void tc_mma_pair(std::uint32_t tmem_d, std::uint64_t adesc,
                                            std::uint64_t bdesc, std::uint32_t idesc,
                                            std::uint32_t accumulate) {
  if constexpr (kTf32) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// Arrive on the cluster leader's copy of a barrier (same smem offset).
__device__ __forceinline__ void mbar_arrive_leader(std::uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

template <bool kTf32, int kStagesT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 float* __restrict__ C, int m, int n, std::uint64_t ldc, int ktiles, int mt, int nt,
                 int group_m) {
  extern __shared__ __align__(1024) std::uint8_t smem_raw[];
  std::uint8_t* smem = reinterpret_cast<std::uint8_t*>(
      (reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~static_cast<std::uintptr_t>(1023));
  std::uint8_t* tiles = smem;
  auto* bars = reinterpret_cast<std::uint64_t*>(smem + kStagesT * kStageBytes2);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + kStagesT;
  std::uint64_t* tmem_full = bars + 2 * kStagesT;
  std::uint64_t* tmem_empty = tmem_full + 2;
  auto* tmem_slot = reinterpret_cast<std::uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const TileMap tm{mt, nt, group_m};  // 256 x 256 tiles
  const int ntiles = mt * nt;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < kStagesT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const std::uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const std::uint32_t a_row0 = rank * 128;
      int stage = 0;
      std::uint32_t phase = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        int mb, nb;
        tm.coords(t, mb, nb);
        for (int kb = 0; kb < ktiles; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          std::uint8_t* sa = tiles + stage * kStageBytes2;
          const std::uint32_t leader_full = smem_u32(&full[stage]) & kPeerMask;
          if (leader) mbar_expect_tx(&full[stage], 2 * kStageBytes2);
          const int kx = kb * (kTf32 ? 32 : 64);
          tma_load_2d_pair(&map_a, leader_full, sa, kx, mb * 256 + a_row0);
          tma_load_2d_pair(&map_b, leader_full, sa + 128 * 128, kx, nb * 256 + a_row0);
          if (++stage == kStagesT) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr std::uint32_t idesc = instr_desc<kTf32, 256, 256>();
      int stage = 0;
      std::uint32_t phase = 0;
      int acc = 0;
      std::uint32_t acc_phase = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const std::uint32_t tmem_d = tmem_base + static_cast<std::uint32_t>(acc * 256);
        for (int kb = 0; kb < ktiles; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const std::uint8_t* sa = tiles + stage * kStageBytes2;
          const std::uint64_t adesc = smem_desc(sa);
          const std::uint64_t bdesc = smem_desc(sa + 128 * 128);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma_pair<kTf32>(tmem_d, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          tc_commit_pair(&empty[stage]);
          if (++stage == kStagesT) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_pair(&tmem_full[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    const int quarter = warp - kEpiWarp0;
    int acc = 0;
    std::uint32_t acc_phase = 0;
    const bool vec_ok = (ldc % 4 == 0) && ((reinterpret_cast<std::uintptr_t>(C) & 15) == 0);
    for (int t = pair; t < ntiles; t += npairs) {
      int mb, nb;
      tm.coords(t, mb, nb);
      mbar_wait_sleepy(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const int row = mb * 256 + static_cast<int>(rank) * 128 + quarter * 32 + lane;
      float* crow = C + static_cast<std::uint64_t>(row) * ldc;
      const std::uint32_t taddr = tmem_base + (static_cast<std::uint32_t>(quarter * 32) << 16) +
                                  static_cast<std::uint32_t>(acc * 256);
#pragma unroll 1
      for (int c = 0; c < 256; c += 32) {
        std::uint32_t v[32];
        tmem_ld32(taddr + c, v);
        const int col = nb * 256 + c;
        if (row < m) {
          if (vec_ok && col + 32 <= n) {
            float4* dst = reinterpret_cast<float4*>(crow + col);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                   __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < n) crow[col + j] = __uint_as_float(v[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tmem_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// ------------------------------------------------------------ operand prep ---

__device__ __forceinline__ float round_tf32(float x) {
  std::uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// 8 operand values -> their prepared form (bf16 RNE: one uint4; tf32 RNA:
// two float4), stored at dst (16-byte aligned).
template <bool kTf32>
__device__ __forceinline__ void store8(void* dst, const float (&x)[8]) {
  if constexpr (kTf32) {
    float4* d = static_cast<float4*>(dst);
    d[0] = make_float4(round_tf32(x[0]), round_tf32(x[1]), round_tf32(x[2]), round_tf32(x[3]));
    d[1] = make_float4(round_tf32(x[4]), round_tf32(x[5]), round_tf32(x[6]), round_tf32(x[7]));
  } else {
    uint4 v;
    std::uint32_t* w = reinterpret_cast<std::uint32_t*>(&v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
      w[j] = *reinterpret_cast<const std::uint32_t*>(&h);
    }
    *static_cast<uint4*>(dst) = v;
  }
}

// A (m x k, lda) -> A' (m x kp), K-major; zero padding beyond k.  One warp
// per row at a time, 8 consecutive values per lane per step (two 128-bit
// loads when A is 16-byte aligned with lda % 4 == 0; one 16- or 32-byte
// store).  HBM-bound: 4 B read + 2 (bf16) / 4 (tf32) B written per value.
template <bool kTf32>
__global__ void __launch_bounds__(256)
    prep_a_kernel(const float* __restrict__ A, std::uint64_t lda, int m, int k, int kp,
                  void* __restrict__ out) {
  constexpr int kEs = kTf32 ? 4 : 2;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * 8;
  const bool vec = ((reinterpret_cast<std::uintptr_t>(A) & 15) == 0) && (lda % 4 == 0);
  const int chunks = kp / 8;
  for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < m; r += warps) {
    const float* src = A + static_cast<std::uint64_t>(r) * lda;
    auto* dst = static_cast<std::uint8_t*>(out) + static_cast<std::uint64_t>(r) * kp * kEs;
    for (int c = lane; c < chunks; c += 32) {
      const int c0 = c * 8;
      float x[8];
      if (vec && c0 + 8 <= k) {
        const float4 p = __ldcs(reinterpret_cast<const float4*>(src + c0));
        const float4 q = __ldcs(reinterpret_cast<const float4*>(src + c0 + 4));
        x[0] = p.x; x[1] = p.y; x[2] = p.z; x[3] = p.w;
        x[4] = q.x; x[5] = q.y; x[6] = q.z; x[7] = q.w;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = c0 + j < k ? src[c0 + j] : 0.f;
      }
      store8<kTf32>(dst + static_cast<std::uint64_t>(c0) * kEs, x);
    }
  }
}

// B (k x n, ldb) -> B'^T (n x kp), K-major.  64 (k) x 64 (n) tile per CTA
// through smem (row pitch 65 floats: conflict-free column reads); loads
// are 128-bit along n, stores 8 consecutive k values (16 / 32 B) per lane,
// 8 lanes per output row = 128 / 256 contiguous bytes.
template <bool kTf32>
__global__ void __launch_bounds__(256)
    prep_bt_kernel(const float* __restrict__ B, std::uint64_t ldb, int k, int n, int kp,
                   void* __restrict__ out) {
  constexpr int kEs = kTf32 ? 4 : 2;
  __shared__ float tile[64][65];
  const int k0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  const int t = threadIdx.x;
  const bool vec = ((reinterpret_cast<std::uintptr_t>(B) & 15) == 0) && (ldb % 4 == 0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = t + 256 * i;           // 1024 float4 slots
    const int kk = idx >> 4, nn = (idx & 15) * 4;
    const int gk = k0 + kk, gn = n0 + nn;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (gk < k) {
      const float* row = B + static_cast<std::uint64_t>(gk) * ldb;
      if (vec && gn + 4 <= n) {
        const float4 p = __ldcs(reinterpret_cast<const float4*>(row + gn));
        v[0] = p.x; v[1] = p.y; v[2] = p.z; v[3] = p.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (gn + j < n) v[j] = row[gn + j];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) tile[kk][nn + j] = v[j];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int idx = t + 256 * i;           // 512 (row, 8-value chunk) slots
    const int nn = idx >> 3, kc = (idx & 7) * 8;
    const int gn = n0 + nn, gk = k0 + kc;
    if (gn < n && gk < kp) {
      float x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = tile[kc + j][nn];
      store8<kTf32>(static_cast<std::uint8_t*>(out) +
                        (static_cast<std::uint64_t>(gn) * kp + gk) * kEs,
                    x);
    }
  }
}

// -------------------------------------------------------------- host side ---

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (fn == nullptr) fail(Errc::TaskFailed, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// rows x kp operand, K-major, box = 128 bytes of K x box_rows rows.
CUtensorMap make_map(void* base, bool tf32, std::uint64_t rows, std::uint64_t kp, int box_rows) {
  CUtensorMap map;
  const std::uint64_t es = tf32 ? 4 : 2;
  const cuuint64_t dims[2] = {kp, rows};
  const cuuint64_t strides[1] = {kp * es};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / es), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&map, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(Errc::TaskFailed, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return map;
}

std::uint64_t k_pad(int prec, std::uint64_t k) {
  const std::uint64_t kt = prec == GPCX_PREC_TF32 ? 32 : 64;
  return (k + kt - 1) / kt * kt;
}

std::uint64_t align256(std::uint64_t x) { return (x + 255) & ~255ull; }

// CTA-pair kernel for problems with enough 256 x 256 tiles to fill the
// SM pairs; the 1-SM 128 x 256 kernel for small / skinny ones.  The
// GPCX_TC_KERNEL=1sm|2sm override exists for tests and A/B measurements.
bool use_pair_kernel(std::uint64_t m, std::uint64_t n, std::uint64_t k, int sms) {
  const char* force = std::getenv("GPCX_TC_KERNEL");
  if (force != nullptr && std::string(force) == "1sm") return false;
  if (force != nullptr && std::string(force) == "2sm") return true;
  // Measured on B200 (tools/c4_ab.py, tools/gemm_sweep.sh, profiles/r1):
  // the pair kernel wins at K <= 8192 (1115 vs 1039 TFLOP/s at 8192^3).
  // With a 7-stage ring it lost at K = 32768 (its CTA pairs drifted apart
  // and their shared panels fell out of L2: 10.6 vs 4.6 GB of DRAM reads
  // on 8192x8192x32768); with the 4-stage ring it runs now it wins there
  // too, so the choice depends on the tile count only, not on K.
  const std::uint64_t tiles2 = ((m + 255) / 256) * ((n + 255) / 256);
  (void)k;
  return m >= 256 && tiles2 >= static_cast<std::uint64_t>(sms / 2);
}

}  // namespace

std::uint64_t tc_workspace_bytes(int prec, std::uint64_t m, std::uint64_t n, std::uint64_t k) {
  const std::uint64_t es = prec == GPCX_PREC_TF32 ? 4 : 2;
  const std::uint64_t kp = k_pad(prec, k);
  return align256(m * kp * es) + align256(n * kp * es);
}

void launch_tc(int prec, std::uint64_t m, std::uint64_t n, std::uint64_t k, const float* A,
               std::uint64_t lda, const float* B, std::uint64_t ldb, float* C, std::uint64_t ldc,
               void* ws, cudaStream_t stream) {
  if (m == 0 || n == 0) return;
  if (m > 0x7FFFFFFFull || n > 0x7FFFFFFFull || k > 0x7FFFFFFFull)
    fail(Errc::TooLarge, "matmul dimension exceeds 2^31");
  if (k == 0) {
    for (std::uint64_t r = 0; r < m; ++r)
      GPCX_CUDA(cudaMemsetAsync(C + r * ldc, 0, n * sizeof(float), stream));
    return;
  }
  const bool tf32 = prec == GPCX_PREC_TF32;
  const std::uint64_t es = tf32 ? 4 : 2;
  const std::uint64_t kp = k_pad(prec, k);
  auto* a_p = static_cast<std::uint8_t*>(ws);
  auto* b_p = a_p + align256(m * kp * es);

  const int sms = device_sm_count();
  {
    const int grid_a = static_cast<int>(std::min<std::uint64_t>((m + 7) / 8, 32ull * sms));
    if (tf32) prep_a_kernel<true><<<grid_a, 256, 0, stream>>>(A, lda, (int)m, (int)k, (int)kp, a_p);
    else prep_a_kernel<false><<<grid_a, 256, 0, stream>>>(A, lda, (int)m, (int)k, (int)kp, a_p);
    GPCX_LAUNCH_CHECK();
    const dim3 g2(static_cast<unsigned>((kp + 63) / 64), static_cast<unsigned>((n + 63) / 64));
    if (g2.y > 65535) fail(Errc::TooLarge, "n too large for the transpose grid");
    if (tf32) prep_bt_kernel<true><<<g2, 256, 0, stream>>>(B, ldb, (int)k, (int)n, (int)kp, b_p);
    else prep_bt_kernel<false><<<g2, 256, 0, stream>>>(B, ldb, (int)k, (int)n, (int)kp, b_p);
    GPCX_LAUNCH_CHECK();
  }

  const int ktiles = static_cast<int>(kp / (tf32 ? 32 : 64));
  if (use_pair_kernel(m, n, k, sms)) {
    const CUtensorMap ma = make_map(a_p, tf32, m, kp, 128);
    const CUtensorMap mb = make_map(b_p, tf32, n, kp, 128);
    const int mt = static_cast<int>((m + 255) / 256), nt = static_cast<int>((n + 255) / 256);
    const int grid = 2 * std::min(mt * nt, sms / 2);
    const char* gs = std::getenv("GPCX_TC_GROUPM");  // A/B knob (tools/, profiles/)
    const int group_m = gs != nullptr ? std::max(1, std::atoi(gs)) : 8;
    const char* ss = std::getenv("GPCX_TC_STAGES2");
    // 4 stages: a deeper ring lets the CTA pairs of a wave drift apart and
    // the shared operand panels fall out of L2 (8192x8192x32768: 4 stages
    // 4.57 GB DRAM reads, 75.6% L2 hits; 7 stages 8.91 GB, 66.8%).
    const int stages = ss != nullptr ? std::atoi(ss) : 4;
    auto go = [&](auto kernel, int smem) {
      GPCX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kernel<<<grid, kThreads, smem, stream>>>(ma, mb, C, (int)m, (int)n, ldc, ktiles, mt, nt, group_m);
    };
    if (tf32) {
      if (stages == 3) go(gemm2_kernel<true, 3>, smem_bytes2<3>());
      else if (stages == 5) go(gemm2_kernel<true, 5>, smem_bytes2<5>());
      else if (stages == 7) go(gemm2_kernel<true, 7>, smem_bytes2<7>());
      else go(gemm2_kernel<true, 4>, smem_bytes2<4>());
    } else {
      if (stages == 3) go(gemm2_kernel<false, 3>, smem_bytes2<3>());
      else if (stages == 5) go(gemm2_kernel<false, 5>, smem_bytes2<5>());
      else if (stages == 7) go(gemm2_kernel<false, 7>, smem_bytes2<7>());
      else go(gemm2_kernel<false, 4>, smem_bytes2<4>());
    }
    GPCX_LAUNCH_CHECK();
    return;
  }
  const CUtensorMap ma = make_map(a_p, tf32, m, kp, BM);
  const CUtensorMap mb = make_map(b_p, tf32, n, kp, BN);
  const int mt = static_cast<int>((m + BM - 1) / BM), nt = static_cast<int>((n + BN - 1) / BN);
  const int grid = std::min(mt * nt, sms);
  if (tf32) {
    GPCX_CUDA(cudaFuncSetAttribute(gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    gemm_kernel<true><<<grid, kThreads, kSmemBytes, stream>>>(ma, mb, C, (int)m, (int)n, ldc, ktiles, mt, nt);
  } else {
    GPCX_CUDA(cudaFuncSetAttribute(gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    gemm_kernel<false><<<grid, kThreads, kSmemBytes, stream>>>(ma, mb, C, (int)m, (int)n, ldc, ktiles, mt, nt);
  }
  GPCX_LAUNCH_CHECK();
}

}  // namespace gpcx::gemm
