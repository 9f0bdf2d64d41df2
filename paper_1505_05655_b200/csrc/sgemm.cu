// sgemm.cu -- FP32-exact SIMT matrix multiply (MATMUL prec=f32).
//
// The reference has no matmul; the task contract is
// SURVEY.md §8a' a'4 with the row-major convention of lsq::Matrix
// (proj/include/gpc/lsq.hpp:34-43).  This is the "FP32-exact SIMT fallback
// kernel when the task demands reference precision" of the north star:
// plain fp32 FFMA accumulation in a fixed, K-ascending order per output, so
// results are deterministic and identical for any block-row sharding.
//
// Tiling: 128x128 CTA tile, BK = 8 or 16, 256 threads each owning an 8x8
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

void launch_sgemm(std::uint64_t m, std::uint64_t n, std::uint64_t k,
                  const float* A, std::uint64_t lda, const float* B,
                  std::uint64_t ldb, float* C, std::uint64_t ldc,
                  cudaStream_t stream) {
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
  // Default BK=8 with 2 CTAs/SM: 49.6 / 50.8 TFLOP/s at 4096^3 / 8192^3 vs
  // 47.4 / 48.5 for BK=16, 1 CTA/SM (B200, tools/mm_micro.py).
  const std::string variant = v != nullptr ? v : "8x2";
  if (variant == "16x1") launch_variant<16, 1>(m, n, k, A, lda, B, ldb, C, ldc, stream);
  else if (variant == "16x2") launch_variant<16, 2>(m, n, k, A, lda, B, ldb, C, ldc, stream);
  else launch_variant<8, 2>(m, n, k, A, lda, B, ldb, C, ldc, stream);
}

}  // namespace gpcx::gemm
