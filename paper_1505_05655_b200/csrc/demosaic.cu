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
// One CTA = a 16 x 256 output tile.  The (16+2) x (256+2) input tile with a
// 1-pixel halo is staged in smem with the edge clamp applied at load time
// (so the stencil is branch-free): interior rows arrive as one 128-bit load
// per lane, the interior starts at a 16-byte aligned smem column, and each
// thread reads its 4 x 10 neighbourhood as 4 x (one 128-bit + two 16-bit)
// smem loads, produces a 2 x 8 block and writes it as 128-bit stores to the
// three planes (R || G || B, each rows*cols u16: the reference's
// rgb_to_le_bytes layout).  HBM-bound: 2 B in + 6 B out per pixel.
#include <cuda_runtime.h>

#include <cstdint>

#include "cuda_util.hpp"
#include "kernels.hpp"

namespace gpcx::demosaic {

namespace {

constexpr int TR = 16, TC = 256, THREADS = 256;
constexpr int kPad = 8;              // smem column of image column c0 (16-byte aligned)
constexpr int SW = kPad + TC + 8;    // row stride in u16 (544 B; rows start 16-byte aligned)

__device__ __forceinline__ std::uint32_t avg2(std::uint32_t a, std::uint32_t b) {
  return (a + b + 1) >> 1;
}
__device__ __forceinline__ std::uint32_t avg4(std::uint32_t a, std::uint32_t b, std::uint32_t c,
                                              std::uint32_t d) {
  return (a + b + c + d + 2) >> 2;
}

// 10 consecutive samples of one smem row: [x0-1, x0+8] around the thread's
// 8 columns starting at smem column x0 (16-byte aligned).
struct Row10 {
  std::uint32_t v[10];
};

__device__ __forceinline__ Row10 load_row(const std::uint16_t* srow, int x0) {
  Row10 r;
  const uint4 q = *reinterpret_cast<const uint4*>(srow + x0);
  r.v[0] = srow[x0 - 1];
  r.v[1] = q.x & 0xFFFFu;
  r.v[2] = q.x >> 16;
  r.v[3] = q.y & 0xFFFFu;
  r.v[4] = q.y >> 16;
  r.v[5] = q.z & 0xFFFFu;
  r.v[6] = q.z >> 16;
  r.v[7] = q.w & 0xFFFFu;
  r.v[8] = q.w >> 16;
  r.v[9] = srow[x0 + 8];
  return r;
}

template <bool kGradient>
__global__ void __launch_bounds__(THREADS, 4)
    demosaic_kernel(const std::uint16_t* __restrict__ in, std::uint16_t* __restrict__ out,
                    int rows, int cols, int dr, int dc, int vec_ok) {
  __shared__ __align__(16) std::uint16_t tile[TR + 2][SW];
  const int r0 = blockIdx.y * TR, c0 = blockIdx.x * TC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Stage the tile: row i of the tile is image row clamp(r0 - 1 + i).
  const bool full_cols = vec_ok && c0 + TC <= cols;
  for (int i = warp; i < TR + 2; i += THREADS / 32) {
    const int gr = min(max(r0 - 1 + i, 0), rows - 1);
    const std::uint16_t* grow = in + static_cast<std::uint64_t>(gr) * cols;
    std::uint16_t* srow = tile[i];
    if (full_cols) {
      reinterpret_cast<uint4*>(srow + kPad)[lane] = reinterpret_cast<const uint4*>(grow + c0)[lane];
    } else {
      for (int c = lane; c < TC; c += 32) srow[kPad + c] = grow[min(c0 + c, cols - 1)];
    }
    if (lane == 0) srow[kPad - 1] = grow[max(c0 - 1, 0)];
    if (lane == 1) srow[kPad + TC] = grow[min(c0 + TC, cols - 1)];
  }
  __syncthreads();

  const std::uint64_t plane = static_cast<std::uint64_t>(rows) * cols;
  const int ty = warp, tx = lane;
  const int x0 = kPad + 8 * tx;
  const int col0 = c0 + 8 * tx;
  if (col0 >= cols) return;
  // rows 2ty-1 .. 2ty+2 of the tile (smem rows 2ty .. 2ty+3)
  const Row10 rw[4] = {load_row(tile[2 * ty], x0), load_row(tile[2 * ty + 1], x0),
                       load_row(tile[2 * ty + 2], x0), load_row(tile[2 * ty + 3], x0)};
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int row = r0 + 2 * ty + rr;
    if (row >= rows) break;
    const Row10& up = rw[rr];
    const Row10& mid = rw[rr + 1];
    const Row10& dn = rw[rr + 2];
    const bool even_row = ((row + dr) & 1) == 0;
    std::uint32_t pr[8], pg[8], pb[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const bool even_col = ((col0 + cc + dc) & 1) == 0;
      const std::uint32_t s = mid.v[cc + 1];
      const std::uint32_t n = up.v[cc + 1], so = dn.v[cc + 1];
      const std::uint32_t w = mid.v[cc], e = mid.v[cc + 2];
      if (even_row == even_col) {  // R (even/even) or B (odd/odd) site
        std::uint32_t g;
        if constexpr (kGradient) {
          const std::uint32_t dh = w > e ? w - e : e - w;
          const std::uint32_t dv = n > so ? n - so : so - n;
          g = dh < dv ? avg2(w, e) : (dv < dh ? avg2(n, so) : avg4(n, so, w, e));
        } else {
          g = avg4(n, so, w, e);
        }
        const std::uint32_t diag = avg4(up.v[cc], up.v[cc + 2], dn.v[cc], dn.v[cc + 2]);
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
    const std::uint64_t off = static_cast<std::uint64_t>(row) * cols + col0;
    if (vec_ok && col0 + 8 <= cols) {
      const uint4 vr = make_uint4(pr[0] | (pr[1] << 16), pr[2] | (pr[3] << 16), pr[4] | (pr[5] << 16),
                                  pr[6] | (pr[7] << 16));
      const uint4 vg = make_uint4(pg[0] | (pg[1] << 16), pg[2] | (pg[3] << 16), pg[4] | (pg[5] << 16),
                                  pg[6] | (pg[7] << 16));
      const uint4 vb = make_uint4(pb[0] | (pb[1] << 16), pb[2] | (pb[3] << 16), pb[4] | (pb[5] << 16),
                                  pb[6] | (pb[7] << 16));
      __stcs(reinterpret_cast<uint4*>(out + off), vr);
      __stcs(reinterpret_cast<uint4*>(out + plane + off), vg);
      __stcs(reinterpret_cast<uint4*>(out + 2 * plane + off), vb);
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
  // 128-bit paths need every row and every plane to start 16-byte aligned.
  const int vec_ok = (cols % 8 == 0) && (plane % 8 == 0) &&
                     (((reinterpret_cast<std::uintptr_t>(out) | reinterpret_cast<std::uintptr_t>(in)) & 15) == 0);
  const dim3 grid(static_cast<unsigned>((cols + TC - 1) / TC), static_cast<unsigned>((rows + TR - 1) / TR));
  if (grid.y > 65535) fail(Errc::TooLarge, "too many rows for the tile grid");
  if (gradient)
    demosaic_kernel<true><<<grid, THREADS, 0, stream>>>(in, out, (int)rows, (int)cols, dr, dc, vec_ok);
  else
    demosaic_kernel<false><<<grid, THREADS, 0, stream>>>(in, out, (int)rows, (int)cols, dr, dc, vec_ok);
  GPCX_LAUNCH_CHECK();
}

}  // namespace gpcx::demosaic
