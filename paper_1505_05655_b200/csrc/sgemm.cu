// sgemm.cu -- FP32-exact SIMT matrix multiply (MATMUL prec=f32).
//
// The reference has no matmul; the task contract is
// SURVEY.md §8a' a'4 with the row-major convention of lsq::Matrix
// (proj/include/gpc/lsq.hpp:34-43).  This is the "FP32-exact SIMT fallback
// kernel when the task demands reference precision" of the north star:
// plain fp32 FFMA accumulation in a fixed, K-ascending order per output, so
// results are deterministic and identical for any block-row sharding.
//
// sgemm4_kernel (aligned shapes, workspace for A^T): the default, see below.
// sgemm2_kernel (aligned shapes, no workspace): cp.async multistage.
// sgemm_kernel (any shape): 128x128 CTA tile, BK = 8 or 16, 256 threads each owning an 8x8
// block (2x2 quads of 4x4 so the 128-bit smem reads stay conflict-free), A
// staged transposed, double-buffered smem with register prefetch of the
// next tile.  Variant <BK, min CTAs/SM> is picked per launch
// (GPCX_SGEMM=16x1|8x2|16x2 overrides, for A/B measurement).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "cuda_util.hpp"
#include "kernels.hpp"

namespace gpcx::gemm {

namespace {

constexpr int BM = 128, BN = 128, THREADS = 256;

template <int BK, int MINB, bool kChecked>
__global__ void __launch_bounds__(THREADS, MINB)
    sgemm_kernel(int m, int n, int k, const float* __restrict__ A,
                 std::uint64_t lda, const float* __restrict__ B,
                 std::uint64_t ldb, float* __restrict__ C, std::uint64_t ldc) {
  constexpr int kLoads = BK / 8;  // float4 of A and of B per thread per tile
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

  float4 ra[kLoads], rb[kLoads];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int i = 0; i < kLoads; ++i) {
      const int f = tid + THREADS * i;
      const int gr = m0 + (f & (BM - 1));
      const int gk = k0 + (f >> 7) * 4;
      if constexpr (!kChecked) {
        ra[i] = *reinterpret_cast<const float4*>(A + static_cast<std::uint64_t>(gr) * lda + gk);
      } else {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[j] = (gr < m && gk + j < k) ? A[static_cast<std::uint64_t>(gr) * lda + gk + j] : 0.f;
        ra[i] = make_float4(v[0], v[1], v[2], v[3]);
      }
      const int bk = k0 + (f >> 5);
      const int bc = n0 + (f & 31) * 4;
      if constexpr (!kChecked) {
        rb[i] = *reinterpret_cast<const float4*>(B + static_cast<std::uint64_t>(bk) * ldb + bc);
      } else {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[j] = (bk < k && bc + j < n) ? B[static_cast<std::uint64_t>(bk) * ldb + bc + j] : 0.f;
        rb[i] = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int i = 0; i < kLoads; ++i) {
      const int f = tid + THREADS * i;
      const int row = f & (BM - 1), k4 = (f >> 7) * 4;
      As[buf][k4 + 0][row] = ra[i].x;
      As[buf][k4 + 1][row] = ra[i].y;
      As[buf][k4 + 2][row] = ra[i].z;
      As[buf][k4 + 3][row] = ra[i].w;
      *reinterpret_cast<float4*>(&Bs[buf][f >> 5][(f & 31) * 4]) = rb[i];
    }
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  const int ktiles = (k + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();

  for (int t = 0; t < ktiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < ktiles) load_tile((t + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4 + 64]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4 + 64]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (t + 1 < ktiles) {
      store_tile(buf ^ 1);
      __syncthreads();
    }
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int gr = m0 + ty * 4 + (i & 3) + (i >> 2) * 64;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gc = n0 + tx * 4 + h * 64;
      float* dst = C + static_cast<std::uint64_t>(gr) * ldc + gc;
      if constexpr (!kChecked) {
        *reinterpret_cast<float4*>(dst) =
            make_float4(acc[i][4 * h], acc[i][4 * h + 1], acc[i][4 * h + 2], acc[i][4 * h + 3]);
      } else {
        if (gr < m) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (gc + j < n) dst[j] = acc[i][4 * h + j];
        }
      }
    }
  }
}

// ---- cp.async multistage variant (aligned shapes) ---------------------
// 128 x 64 CTA tile, 128 threads, 8 x 8 outputs per thread, BK = 16, a
// 3-stage cp.async ring: both operand tiles are copied global -> smem
// without passing through registers, so the K loop issues only LDS + FFMA.
// A stays row-major in smem (row pitch 20 floats): a thread reads its 8
// rows' 4 consecutive k as one LDS.128 each; thread (tx, ty) owns rows
// ty + 16 i (a warp's 4 ty values hit 4 distinct bank groups) and columns
// 4 tx + {0..3}, 32 + 4 tx + {0..3}.  Per 4 k: 16 LDS.128 for 256 FFMA.
// Each output is still fma-accumulated over k in ascending order, so the
// result is bitwise identical to sgemm_kernel's.
constexpr int BM2 = 128, BN2 = 64, THREADS2 = 128;

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<std::uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}

template <int BK2, int STAGES2>
constexpr int sgemm2_smem() {
  return STAGES2 * (BM2 * (BK2 + 4) + BK2 * BN2) * 4;
}

template <int BK2, int STAGES2, int MINB>
__global__ void __launch_bounds__(THREADS2, MINB)
    sgemm2_kernel(int k, const float* __restrict__ A, std::uint64_t lda,
                  const float* __restrict__ B, std::uint64_t ldb, float* __restrict__ C,
                  std::uint64_t ldc) {
  constexpr int APITCH = BK2 + 4;  // floats
  extern __shared__ __align__(16) float smem2[];
  float (*As)[BM2 * APITCH] = reinterpret_cast<float (*)[BM2 * APITCH]>(smem2);
  float (*Bs)[BK2 * BN2] = reinterpret_cast<float (*)[BK2 * BN2]>(smem2 + STAGES2 * BM2 * APITCH);
  const int tid = threadIdx.x;
  const int tx = tid & 7, ty = tid >> 3;
  const int m0 = blockIdx.y * BM2, n0 = blockIdx.x * BN2;
  const float* Ablk = A + static_cast<std::uint64_t>(m0) * lda;
  const float* Bblk = B + n0;

  auto issue = [&](int stage, int k0) {
#pragma unroll
    for (int i = 0; i < BK2 / 4; ++i) {  // A: 128 rows x BK2/4 chunks of 16 B
      const int c = tid + THREADS2 * i;
      const int row = c / (BK2 / 4), q = c % (BK2 / 4);
      cp16(&As[stage][row * APITCH + 4 * q], Ablk + static_cast<std::uint64_t>(row) * lda + k0 + 4 * q);
    }
#pragma unroll
    for (int i = 0; i < BK2 / 8; ++i) {  // B: BK2 rows x 16 chunks of 16 B
      const int c = tid + THREADS2 * i;
      const int kr = c >> 4, q = c & 15;
      cp16(&Bs[stage][kr * BN2 + 4 * q], Bblk + static_cast<std::uint64_t>(k0 + kr) * ldb + 4 * q);
    }
  };

  // acc[i][p] = outputs (row i, columns 2p, 2p+1 of the thread's 8):
  // FFMA2 (Blackwell packed fp32x2 FMA, IEEE fma per lane -> the same bits
  // as two fmaf) with a[i] broadcast: half the FMA instructions and half
  // the accumulator register reads per flop of a scalar FFMA loop.
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 4; ++p) acc[i][p] = make_float2(0.f, 0.f);

  const int ktiles = k / BK2;
#pragma unroll
  for (int st = 0; st < STAGES2 - 1; ++st) {
    if (st < ktiles) issue(st, st * BK2);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int t = 0; t < ktiles; ++t) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES2 - 2) : "memory");
    __syncthreads();  // tile t visible; stage (t - 1) % S free to refill
    const int nt = t + STAGES2 - 1;
    if (nt < ktiles) issue(nt % STAGES2, nt * BK2);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* as = As[t % STAGES2];
    const float* bs = Bs[t % STAGES2];
#pragma unroll
    for (int kq = 0; kq < BK2; kq += 4) {
      float a[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 v = *reinterpret_cast<const float4*>(&as[(ty + 16 * i) * APITCH + kq]);
        a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const float4 b0 = *reinterpret_cast<const float4*>(&bs[(kq + kk) * BN2 + 4 * tx]);
        const float4 b1 = *reinterpret_cast<const float4*>(&bs[(kq + kk) * BN2 + 32 + 4 * tx]);
        const float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w),
                             make_float2(b1.x, b1.y), make_float2(b1.z, b1.w)};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 ai = make_float2(a[i][kk], a[i][kk]);
#pragma unroll
          for (int p = 0; p < 4; ++p) acc[i][p] = __ffma2_rn(ai, b[p], acc[i][p]);
        }
      }
    }
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float* crow = C + static_cast<std::uint64_t>(m0 + ty + 16 * i) * ldc + n0;
    *reinterpret_cast<float4*>(crow + 4 * tx) =
        make_float4(acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y);
    *reinterpret_cast<float4*>(crow + 32 + 4 * tx) =
        make_float4(acc[i][2].x, acc[i][2].y, acc[i][3].x, acc[i][3].y);
  }
}

// ---- A-transposed multistage variant (aligned shapes, with workspace) ---
// A is transposed once into the workspace (At = A^T, k x m, a 64 x 64 smem
// transpose: 2 x m x k x 4 bytes of HBM traffic, ~1% of the 4096^3 GEMM),
// so both operands are MN-major: As[k][m] and Bs[k][n] arrive by 16-byte
// cp.async with coalesced rows, and per k a thread reads 2 + 2 LDS.128
// (rows 4 tm + {0..3} and 64 + 4 tm + {0..3}, columns 4 tn + {0..3} and
// 32 + 4 tn + {0..3}: 64 B of A and 128 B of B per warp, one wavefront
// each) feeding 32 FFMA2.  Against sgemm2_kernel (A row-major, 8 LDS.128
// per 4 k over 8 rows) the fragments of one k need 4 loads instead of 10,
// so the FFMA2 stream starts sooner after each load: 4096^3 53.9 -> 60.0
// TFLOP/s incl. the transpose (B200, tools/mm_micro.py).  Per output the
// fma order is still k ascending: bitwise equal to the other kernels.
__global__ void __launch_bounds__(256)
    transpose_kernel(const float* __restrict__ A, std::uint64_t lda, std::uint64_t m,
                     float* __restrict__ At) {
  // 64 x 64 tile, 16-byte loads and stores (4 of each per thread in flight)
  __shared__ float t[64][65];
  const std::uint64_t k0 = static_cast<std::uint64_t>(blockIdx.x) * 64;
  const std::uint64_t m0 = static_cast<std::uint64_t>(blockIdx.y) * 64;
  const int r = threadIdx.x >> 4, c4 = (threadIdx.x & 15) * 4;
  float4 v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    v[i] = *reinterpret_cast<const float4*>(A + (m0 + r + 16 * i) * lda + k0 + c4);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    t[r + 16 * i][c4 + 0] = v[i].x;
    t[r + 16 * i][c4 + 1] = v[i].y;
    t[r + 16 * i][c4 + 2] = v[i].z;
    t[r + 16 * i][c4 + 3] = v[i].w;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int kr = r + 16 * i;  // row of At (a k), columns m0 + c4 .. + 3
    *reinterpret_cast<float4*>(At + (k0 + kr) * m + m0 + c4) =
        make_float4(t[c4 + 0][kr], t[c4 + 1][kr], t[c4 + 2][kr], t[c4 + 3][kr]);
  }
}

template <int BK4, int STAGES4>
constexpr int sgemm4_smem() {
  return STAGES4 * BK4 * (BM2 + BN2) * 4;
}

template <int BK4, int STAGES4, int MINB>
__global__ void __launch_bounds__(THREADS2, MINB)
    sgemm4_kernel(int m, int k, const float* __restrict__ At, const float* __restrict__ B,
                  std::uint64_t ldb, float* __restrict__ C, std::uint64_t ldc) {
  extern __shared__ __align__(16) float smem4[];
  float (*As)[BK4 * BM2] = reinterpret_cast<float (*)[BK4 * BM2]>(smem4);
  float (*Bs)[BK4 * BN2] = reinterpret_cast<float (*)[BK4 * BN2]>(smem4 + STAGES4 * BK4 * BM2);
  const int tid = threadIdx.x;
  const int tn = tid & 7, tm = tid >> 3;
  const int m0 = blockIdx.y * BM2, n0 = blockIdx.x * BN2;
  auto issue = [&](int stage, int k0) {
#pragma unroll
    for (int i = 0; i < BK4 / 4; ++i) {  // A^T: BK4 k-rows x 32 chunks of 16 B
      const int c = tid + THREADS2 * i;
      const int kr = c >> 5, q = c & 31;
      cp16(&As[stage][kr * BM2 + 4 * q],
           At + static_cast<std::uint64_t>(k0 + kr) * static_cast<std::uint64_t>(m) + m0 + 4 * q);
    }
#pragma unroll
    for (int i = 0; i < BK4 / 8; ++i) {  // B: BK4 k-rows x 16 chunks of 16 B
      const int c = tid + THREADS2 * i;
      const int kr = c >> 4, q = c & 15;
      cp16(&Bs[stage][kr * BN2 + 4 * q], B + static_cast<std::uint64_t>(k0 + kr) * ldb + n0 + 4 * q);
    }
  };
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 4; ++p) acc[i][p] = make_float2(0.f, 0.f);
  const int ktiles = k / BK4;
#pragma unroll
  for (int st = 0; st < STAGES4 - 1; ++st) {
    if (st < ktiles) issue(st, st * BK4);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int t = 0; t < ktiles; ++t) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES4 - 2) : "memory");
    __syncthreads();  // tile t visible; stage (t - 1) % S free to refill
    const int nt = t + STAGES4 - 1;
    if (nt < ktiles) issue(nt % STAGES4, nt * BK4);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* as = As[t % STAGES4];
    const float* bs = Bs[t % STAGES4];
#pragma unroll
    for (int kk = 0; kk < BK4; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&as[kk * BM2 + 4 * tm]);
      const float4 a1 = *reinterpret_cast<const float4*>(&as[kk * BM2 + 64 + 4 * tm]);
      const float4 b0 = *reinterpret_cast<const float4*>(&bs[kk * BN2 + 4 * tn]);
      const float4 b1 = *reinterpret_cast<const float4*>(&bs[kk * BN2 + 32 + 4 * tn]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 b[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w),
                           make_float2(b1.x, b1.y), make_float2(b1.z, b1.w)};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 ai = make_float2(a[i], a[i]);
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[i][p] = __ffma2_rn(ai, b[p], acc[i][p]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = m0 + (i < 4 ? 4 * tm + i : 64 + 4 * tm + (i - 4));
    float* crow = C + static_cast<std::uint64_t>(row) * ldc + n0;
    *reinterpret_cast<float4*>(crow + 4 * tn) =
        make_float4(acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y);
    *reinterpret_cast<float4*>(crow + 32 + 4 * tn) =
        make_float4(acc[i][2].x, acc[i][2].y, acc[i][3].x, acc[i][3].y);
  }
}

bool sgemm2_fits(std::uint64_t m, std::uint64_t n, std::uint64_t k, const float* A,
                 std::uint64_t lda, const float* B, std::uint64_t ldb, const float* C,
                 std::uint64_t ldc) {
  return m % BM2 == 0 && n % BN2 == 0 && k % 32 == 0 && lda % 4 == 0 && ldb % 4 == 0 &&
         ldc % 4 == 0 && (m / BM2) <= 65535 &&
         ((reinterpret_cast<std::uintptr_t>(A) | reinterpret_cast<std::uintptr_t>(B) |
           reinterpret_cast<std::uintptr_t>(C)) & 15u) == 0;
}

template <int BK, int MINB>
void launch_variant(std::uint64_t m, std::uint64_t n, std::uint64_t k, const float* A,
                    std::uint64_t lda, const float* B, std::uint64_t ldb, float* C,
                    std::uint64_t ldc, cudaStream_t stream) {
  const dim3 grid(static_cast<unsigned>((n + BN - 1) / BN), static_cast<unsigned>((m + BM - 1) / BM));
  const bool aligned =
      m % BM == 0 && n % BN == 0 && k % BK == 0 && lda % 4 == 0 && ldb % 4 == 0 &&
      ldc % 4 == 0 &&
      ((reinterpret_cast<std::uintptr_t>(A) | reinterpret_cast<std::uintptr_t>(B) |
        reinterpret_cast<std::uintptr_t>(C)) & 15u) == 0;
  if (aligned)
    sgemm_kernel<BK, MINB, false><<<grid, THREADS, 0, stream>>>(
        static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), A, lda, B, ldb, C, ldc);
  else
    sgemm_kernel<BK, MINB, true><<<grid, THREADS, 0, stream>>>(
        static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), A, lda, B, ldb, C, ldc);
  GPCX_LAUNCH_CHECK();
}

}  // namespace

std::uint64_t sgemm_workspace_bytes(std::uint64_t m, std::uint64_t n, std::uint64_t k) {
  // A^T for sgemm4_kernel (aligned shapes; the pointers are checked at launch)
  const bool shape_ok = m % BM2 == 0 && n % BN2 == 0 && k % 64 == 0 && m > 0 && n > 0 &&
                        m <= 0x7FFFFFFFull && k <= 0x7FFFFFFFull && (m / BM2) <= 65535;
  return shape_ok ? m * k * 4 : 0;
}

void launch_sgemm(std::uint64_t m, std::uint64_t n, std::uint64_t k,
                  const float* A, std::uint64_t lda, const float* B,
                  std::uint64_t ldb, float* C, std::uint64_t ldc,
                  void* ws, std::uint64_t ws_bytes, cudaStream_t stream) {
  if (m == 0 || n == 0) return;
  if (m > 0x7FFFFFFFull || n > 0x7FFFFFFFull || k > 0x7FFFFFFFull)
    fail(Errc::TooLarge, "matmul dimension exceeds 2^31");
  if ((m + BM - 1) / BM > 65535) fail(Errc::TooLarge, "m too large for the SIMT grid");
  if (k == 0) {
    for (std::uint64_t r = 0; r < m; ++r)
      GPCX_CUDA(cudaMemsetAsync(C + r * ldc, 0, n * sizeof(float), stream));
    return;
  }
  const char* v = std::getenv("GPCX_SGEMM");
  const std::string variant = v != nullptr ? v : "";
  const std::uint64_t at_bytes = sgemm_workspace_bytes(m, n, k);
  if ((variant.empty() || variant[0] == 't') && at_bytes != 0 && ws != nullptr &&
      ws_bytes >= at_bytes && (reinterpret_cast<std::uintptr_t>(ws) & 15u) == 0 &&
      sgemm2_fits(m, n, k, A, lda, B, ldb, C, ldc)) {
    auto* at = static_cast<float*>(ws);
    transpose_kernel<<<dim3(static_cast<unsigned>(k / 64), static_cast<unsigned>(m / 64)), 256, 0,
                       stream>>>(A, lda, m, at);
    GPCX_LAUNCH_CHECK();
    const dim3 grid(static_cast<unsigned>(n / BN2), static_cast<unsigned>(m / BM2));
    auto go = [&](auto kernel, int smem) {
      GPCX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kernel<<<grid, THREADS2, smem, stream>>>(static_cast<int>(m), static_cast<int>(k), at, B,
                                               ldb, C, ldc);
    };
    // GPCX_SGEMM=t32x3 | t16x4 for A/B runs
    if (variant == "t32x3") go(sgemm4_kernel<32, 3, 2>, sgemm4_smem<32, 3>());
    else if (variant == "t16x4") go(sgemm4_kernel<16, 4, 2>, sgemm4_smem<16, 4>());
    else go(sgemm4_kernel<16, 3, 2>, sgemm4_smem<16, 3>());
    GPCX_LAUNCH_CHECK();
    return;
  }
  // no workspace (or GPCX_SGEMM=c...): A read row-major by sgemm2_kernel
  if ((variant.empty() || variant[0] == 'c' || variant[0] == 't') &&
      sgemm2_fits(m, n, k, A, lda, B, ldb, C, ldc)) {
    const dim3 grid(static_cast<unsigned>(n / BN2), static_cast<unsigned>(m / BM2));
    auto go = [&](auto kernel, int smem) {
      GPCX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kernel<<<grid, THREADS2, smem, stream>>>(static_cast<int>(k), A, lda, B, ldb, C, ldc);
    };
    // GPCX_SGEMM=c16x3 | c16x4 | c32x3 (BK x stages) for A/B runs
    if (variant == "c16x4") go(sgemm2_kernel<16, 4, 2>, sgemm2_smem<16, 4>());
    else if (variant == "c32x3") go(sgemm2_kernel<32, 3, 2>, sgemm2_smem<32, 3>());
    else if (variant == "c16x3b3") go(sgemm2_kernel<16, 3, 3>, sgemm2_smem<16, 3>());
    else go(sgemm2_kernel<16, 3, 2>, sgemm2_smem<16, 3>());
    GPCX_LAUNCH_CHECK();
    return;
  }
  // Register-staged kernel for ragged / unaligned shapes (and A/B runs):
  // BK=8 with 2 CTAs/SM: 49.6 / 50.8 TFLOP/s at 4096^3 / 8192^3 vs 47.4 /
  // 48.5 for BK=16, 1 CTA/SM (B200, tools/mm_micro.py).
  if (variant == "16x1") launch_variant<16, 1>(m, n, k, A, lda, B, ldb, C, ldc, stream);
  else if (variant == "16x2") launch_variant<16, 2>(m, n, k, A, lda, B, ldb, C, ldc, stream);
  else launch_variant<8, 2>(m, n, k, A, lda, B, ldb, C, ldc, stream);
}

}  // namespace gpcx::gemm
