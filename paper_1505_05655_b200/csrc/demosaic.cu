// demosaic.cu -- BAYER_BILINEAR / BAYER_GRADIENT on sm_100a (SURVEY.md §8f,
// first "next" row): the reference's per-pixel integer rules
// (proj/src/demosaic.cpp:26-129, proj/include/gpc/demosaic.hpp:14-28), bit-exact:
//
//   R site:          G = avg4(N,S,E,W)  B = avg4(diagonals)
//   B site:          G = avg4(N,S,E,W)  R = avg4(diagonals)
//   G in a red row:  R = avg2(E,W)      B = avg2(N,S)
//   G in a blue row: R = avg2(N,S)      B = avg2(E,W)
//   gradient:        G at R/B = avg2 of the pair with the smaller |difference|,
//                    avg4 on a tie
//   avg2 = (a+b+1)/2, avg4 = (a+b+c+d+2)/4 (round half up), off-image
//   neighbours clamp to the nearest edge pixel (Accessor, demosaic.cpp:26-35),
//   CFA phase = (row, col) shift of the RGGB tile (demosaic.cpp:15-24,151-157).
//
// One CTA = a 16 x 256 output tile: the (16+2) x (256+2) input tile with a
// 1-pixel halo is staged in smem with the edge clamp applied at load time,
// so the stencil itself is branch-free; each thread produces a 2 x 8 block
// and writes it as 128-bit stores to the three planes (R || G || B, each
// rows*cols u16, the reference's rgb_to_le_bytes layout).  HBM-bound:
// 2 B in + 6 B out per pixel.
#include <cuda_runtime.h>

#include <cstdint>

#include "cuda_util.hpp"
#include "kernels.hpp"

namespace gpcx::demosaic {

namespace {

constexpr int TR = 16, TC = 256, THREADS = 256;
constexpr int SW = TC + 2 + 2;  // smem row stride (u16), +2 keeps rows 4-byte aligned

__device__ __forceinline__ std::uint32_t avg2(std::uint32_t a, std::uint32_t b) {
  return (a + b + 1) >> 1;
}
__device__ __forceinline__ std::uint32_t avg4(std::uint32_t a, std::uint32_t b, std::uint32_t c,
                                              std::uint32_t d) {
  return (a + b + c + d + 2) >> 2;
}

template <bool kGradient>
__global__ void __launch_bounds__(THREADS)
    demosaic_kernel(const std::uint16_t* __restrict__ in, std::uint16_t* __restrict__ out,
                    int rows, int cols, int dr, int dc, int vec_ok) {
  __shared__ std::uint16_t tile[TR + 2][SW];
  const int r0 = blockIdx.y * TR, c0 = blockIdx.x * TC;
  for (int idx = threadIdx.x; idx < (TR + 2) * (TC + 2); idx += THREADS) {
    const int r = idx / (TC + 2), c = idx - r * (TC + 2);
    const int gr = min(max(r0 - 1 + r, 0), rows - 1);
    const int gc = min(max(c0 - 1 + c, 0), cols - 1);
    tile[r][c] = in[static_cast<std::uint64_t>(gr) * cols + gc];
  }
  __syncthreads();

  const std::uint64_t plane = static_cast<std::uint64_t>(rows) * cols;
  const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = 2 * ty + rr;  // tile row
    const int row = r0 + r;
    if (row >= rows) continue;
    const bool even_row = ((row + dr) & 1) == 0;
    std::uint32_t pr[8], pg[8], pb[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int c = 8 * tx + cc;
      const int col = c0 + c;
      const bool even_col = ((col + dc) & 1) == 0;
      const std::uint32_t s = tile[r + 1][c + 1];
      const std::uint32_t n = tile[r][c + 1], so = tile[r + 2][c + 1];
      const std::uint32_t w = tile[r + 1][c], e = tile[r + 1][c + 2];
      if (even_row == even_col) {  // R (even/even) or B (odd/odd) site
        std::uint32_t g;
        if constexpr (kGradient) {
          const std::uint32_t dh = w > e ? w - e : e - w;
          const std::uint32_t dv = n > so ? n - so : so - n;
          g = dh < dv ? avg2(w, e) : (dv < dh ? avg2(n, so) : avg4(n, so, w, e));
        } else {
          g = avg4(n, so, w, e);
        }
        const std::uint32_t diag = avg4(tile[r][c], tile[r][c + 2], tile[r + 2][c], tile[r + 2][c + 2]);
        pg[cc] = g;
        pr[cc] = even_row ? s : diag;
        pb[cc] = even_row ? diag : s;
      } else {
        pg[cc] = s;
        const std::uint32_t ew = avg2(w, e), ns = avg2(n, so);
        pr[cc] = even_row ? ew : ns;  // G in a red row: R from E/W
        pb[cc] = even_row ? ns : ew;
      }
    }
    const int col0 = c0 + 8 * tx;
    const std::uint64_t off = static_cast<std::uint64_t>(row) * cols + col0;
    if (vec_ok && col0 + 8 <= cols) {
      const uint4 vr = make_uint4(pr[0] | (pr[1] << 16), pr[2] | (pr[3] << 16), pr[4] | (pr[5] << 16),
                                  pr[6] | (pr[7] << 16));
      const uint4 vg = make_uint4(pg[0] | (pg[1] << 16), pg[2] | (pg[3] << 16), pg[4] | (pg[5] << 16),
                                  pg[6] | (pg[7] << 16));
      const uint4 vb = make_uint4(pb[0] | (pb[1] << 16), pb[2] | (pb[3] << 16), pb[4] | (pb[5] << 16),
                                  pb[6] | (pb[7] << 16));
      *reinterpret_cast<uint4*>(out + off) = vr;
      *reinterpret_cast<uint4*>(out + plane + off) = vg;
      *reinterpret_cast<uint4*>(out + 2 * plane + off) = vb;
    } else {
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        if (col0 + cc >= cols) break;
        out[off + cc] = static_cast<std::uint16_t>(pr[cc]);
        out[plane + off + cc] = static_cast<std::uint16_t>(pg[cc]);
        out[2 * plane + off + cc] = static_cast<std::uint16_t>(pb[cc]);
      }
    }
  }
}

}  // namespace

void launch(bool gradient, int phase, const std::uint16_t* in, std::uint16_t* out,
            std::uint64_t rows, std::uint64_t cols, cudaStream_t stream) {
  if (rows < 2 || cols < 2)
    fail(Errc::BadImage, "image is " + std::to_string(rows) + "x" + std::to_string(cols) +
                             ", need at least 2x2");
  if (rows > 0x7FFFFFFFull || cols > 0x7FFFFFFFull) fail(Errc::TooLarge, "image too large");
  // phase: 0 RGGB (0,0), 1 BGGR (1,1), 2 GRBG (0,1), 3 GBRG (1,0)
  static const int kDr[4] = {0, 1, 0, 1}, kDc[4] = {0, 1, 1, 0};
  const int dr = kDr[phase & 3], dc = kDc[phase & 3];
  const std::uint64_t plane = rows * cols;
  const int vec_ok = (cols % 8 == 0) && (plane % 8 == 0) &&
                     ((reinterpret_cast<std::uintptr_t>(out) & 15) == 0);
  const dim3 grid(static_cast<unsigned>((cols + TC - 1) / TC), static_cast<unsigned>((rows + TR - 1) / TR));
  if (grid.y > 65535) fail(Errc::TooLarge, "too many rows for the tile grid");
  if (gradient)
    demosaic_kernel<true><<<grid, THREADS, 0, stream>>>(in, out, (int)rows, (int)cols, dr, dc, vec_ok);
  else
    demosaic_kernel<false><<<grid, THREADS, 0, stream>>>(in, out, (int)rows, (int)cols, dr, dc, vec_ok);
  GPCX_LAUNCH_CHECK();
}

}  // namespace gpcx::demosaic
