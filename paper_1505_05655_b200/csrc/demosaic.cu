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
// One CTA = an (8 * RPT) x 256 output tile, 256 threads (8 warps x 32
// lanes), RPT = 4 rows per thread for bilinear, 8 for gradient.  The tile
// plus a 1-pixel halo is staged in smem with the edge clamp applied at load
// time (so the stencil is branch-free): each warp issues all of its rows'
// 128-bit loads (and the halo columns) before its first smem store, so a CTA
// has its whole input tile in flight at once.  The interior starts at a
// 16-byte aligned smem column; a thread walks down its 8 columns reading one
// smem row (one 128-bit + two 16-bit loads) per output row, keeps a 3-row
// window in registers, and writes each output row as three 128-bit
// streaming stores to the planes (R || G || B, each rows*cols u16: the
// reference's rgb_to_le_bytes layout).  Site types are compile-time: the
// kernel is specialised on the CFA column phase, and row parity is
// warp-uniform, so no per-pixel select between the formulas remains.
// HBM-bound: 2 B in + 6 B out per pixel.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "cuda_util.hpp"
#include "kernels.hpp"

namespace gpcx::demosaic {

namespace {

constexpr int TC = 256, THREADS = 256;
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

// One output row of the thread's 8 columns.  The site type of column cc is
// compile-time (kDc = column phase, kEvenRow = row phase; col0 is a multiple
// of 8), so each variant carries only its own arithmetic -- no per-pixel
// select between the R/B-site and G-site formulas.
template <bool kGradient, bool kEvenRow, int kDc>
__device__ __forceinline__ void mosaic_row(const Row10& up, const Row10& mid, const Row10& dn,
                                           std::uint32_t (&pr)[8], std::uint32_t (&pg)[8],
                                           std::uint32_t (&pb)[8]) {
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) {
    const bool even_col = ((cc + kDc) & 1) == 0;
    const std::uint32_t s = mid.v[cc + 1];
    const std::uint32_t n = up.v[cc + 1], so = dn.v[cc + 1];
    const std::uint32_t w = mid.v[cc], e = mid.v[cc + 2];
    if (kEvenRow == even_col) {  // R (even/even) or B (odd/odd) site
      std::uint32_t g;
      if constexpr (kGradient) {
        // avg2(x, y) = (2(x + y) + 2) >> 2, so the three candidates share
        // one shift: pick the numerator, then g = t >> 2.
        const std::uint32_t dh = w > e ? w - e : e - w;
        const std::uint32_t dv = n > so ? n - so : so - n;
        const std::uint32_t sh = w + e, sv = n + so;
        const std::uint32_t t = dh < dv ? 2 * sh : (dv < dh ? 2 * sv : sh + sv);
        g = (t + 2) >> 2;
      } else {
        g = avg4(n, so, w, e);
      }
      const std::uint32_t diag = avg4(up.v[cc], up.v[cc + 2], dn.v[cc], dn.v[cc + 2]);
      pg[cc] = g;
      pr[cc] = kEvenRow ? s : diag;
      pb[cc] = kEvenRow ? diag : s;
    } else {
      pg[cc] = s;
      const std::uint32_t ew = avg2(w, e), ns = avg2(n, so);
      pr[cc] = kEvenRow ? ew : ns;  // G in a red row: R from E/W
      pb[cc] = kEvenRow ? ns : ew;
    }
  }
}

__device__ __forceinline__ uint4 pack8(const std::uint32_t (&p)[8]) {
  return make_uint4(__byte_perm(p[0], p[1], 0x5410), __byte_perm(p[2], p[3], 0x5410),
                    __byte_perm(p[4], p[5], 0x5410), __byte_perm(p[6], p[7], 0x5410));
}

// RPT output rows per thread: a CTA covers TR = 8 * RPT rows x 256 columns.
template <int RPT>
constexpr int kMinBlocks = 4;

// A band of output rows [row_base, row_base + out_rows) of a rows x cols
// mosaic: `in` holds image rows [in_row0, ...) (the band plus its 1-row
// halo, or the whole image), `out` three band-local planes of out_rows x
// cols.  Edge clamp and CFA parity use image coordinates, so a band equals
// the same rows of the whole-image result.
template <bool kGradient, int kDc, int RPT, bool kBand>
__global__ void __launch_bounds__(THREADS, kMinBlocks<RPT>)
    demosaic_kernel(const std::uint16_t* __restrict__ in, std::uint16_t* __restrict__ out,
                    int rows, int cols, int dr, int vec_ok, int band_row_base, int band_in_row0,
                    int band_out_rows) {
  // whole image (kBand false): the band arguments fold to constants, so the
  // hot single-device kernel keeps its register budget (64, no spills)
  const int row_base = kBand ? band_row_base : 0;
  const int in_row0 = kBand ? band_in_row0 : 0;
  const int out_rows = kBand ? band_out_rows : rows;
  constexpr int TR = 8 * RPT;
  __shared__ __align__(16) std::uint16_t tile[TR + 2][SW];
  const int r0 = row_base + blockIdx.y * TR, c0 = blockIdx.x * TC;
  const int row_end = row_base + out_rows;
  // last image row staged for this band: its halo row below (row_end) or
  // the image's last row -- a band's last tile may reach past its rows,
  // whose outputs are skipped, and must not read past the band's buffer
  const int last_row = min(rows - 1, row_end);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Stage the tile: row i of the tile is image row clamp(r0 - 1 + i).
  // A warp owns tile rows warp, warp + 8, warp + 16: all of its global loads
  // (rows and halo columns) are issued before the first smem store, so they
  // are in flight together.
  constexpr int kRowsPerWarp = (TR + 2 + THREADS / 32 - 1) / (THREADS / 32);
  constexpr int kBatch = 5;  // rows in flight per warp (64-row tiles: 5 + 4)
  const bool full_cols = vec_ok && c0 + TC <= cols;
  if (full_cols) {
#pragma unroll
    for (int j0 = 0; j0 < kRowsPerWarp; j0 += kBatch) {
      uint4 q[kBatch];
      std::uint32_t halo[kBatch];
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        const int i = warp + (j0 + j) * (THREADS / 32);
        if (j0 + j < kRowsPerWarp && i < TR + 2) {
          const int gr = min(max(r0 - 1 + i, 0), last_row);
          const std::uint16_t* grow = in + static_cast<std::uint64_t>(gr - in_row0) * cols;
          q[j] = __ldg(reinterpret_cast<const uint4*>(grow + c0) + lane);
          if (lane < 2) halo[j] = __ldg(grow + (lane == 0 ? max(c0 - 1, 0) : min(c0 + TC, cols - 1)));
        }
      }
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        const int i = warp + (j0 + j) * (THREADS / 32);
        if (j0 + j < kRowsPerWarp && i < TR + 2) {
          reinterpret_cast<uint4*>(tile[i] + kPad)[lane] = q[j];
          if (lane < 2) tile[i][lane == 0 ? kPad - 1 : kPad + TC] = static_cast<std::uint16_t>(halo[j]);
        }
      }
    }
  } else {
    for (int i = warp; i < TR + 2; i += THREADS / 32) {
      const int gr = min(max(r0 - 1 + i, 0), last_row);
      const std::uint16_t* grow = in + static_cast<std::uint64_t>(gr - in_row0) * cols;
      std::uint16_t* srow = tile[i];
      for (int c = lane; c < TC; c += 32) srow[kPad + c] = grow[min(c0 + c, cols - 1)];
      if (lane == 0) srow[kPad - 1] = grow[max(c0 - 1, 0)];
      if (lane == 1) srow[kPad + TC] = grow[min(c0 + TC, cols - 1)];
    }
  }
  __syncthreads();

  const std::uint64_t plane = static_cast<std::uint64_t>(out_rows) * cols;
  const int ty = warp, tx = lane;
  const int x0 = kPad + 8 * tx;
  const int col0 = c0 + 8 * tx;
  if (col0 >= cols) return;
  // image rows RPT*ty-1 .. RPT*ty+RPT of the tile (smem rows RPT*ty ..
  // RPT*ty+RPT+1); each further row is read after the previous output row
  // is stored (fewer live registers).
  Row10 rw[RPT + 2];
  rw[0] = load_row(tile[RPT * ty], x0);
  rw[1] = load_row(tile[RPT * ty + 1], x0);
  rw[2] = load_row(tile[RPT * ty + 2], x0);
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const int row = r0 + RPT * ty + rr;
    if (row >= row_end) break;
    if (rr >= 1) rw[rr + 2] = load_row(tile[RPT * ty + rr + 2], x0);
    std::uint32_t pr[8], pg[8], pb[8];
    // row parity is warp-uniform (a warp owns one row pair)
    if (((row + dr) & 1) == 0)
      mosaic_row<kGradient, true, kDc>(rw[rr], rw[rr + 1], rw[rr + 2], pr, pg, pb);
    else
      mosaic_row<kGradient, false, kDc>(rw[rr], rw[rr + 1], rw[rr + 2], pr, pg, pb);
    const std::uint64_t off = static_cast<std::uint64_t>(row - row_base) * cols + col0;
    if (vec_ok && col0 + 8 <= cols) {
      __stcs(reinterpret_cast<uint4*>(out + off), pack8(pr));
      __stcs(reinterpret_cast<uint4*>(out + plane + off), pack8(pg));
      __stcs(reinterpret_cast<uint4*>(out + 2 * plane + off), pack8(pb));
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

void launch_band(bool gradient, int phase, const std::uint16_t* in, std::uint16_t* out,
                 std::uint64_t rows, std::uint64_t cols, std::uint64_t row_base,
                 std::uint64_t in_row0, std::uint64_t out_rows, cudaStream_t stream) {
  if (rows < 2 || cols < 2)
    fail(Errc::BadImage, "image is " + std::to_string(rows) + "x" + std::to_string(cols) +
                             ", need at least 2x2");
  if (rows > 0x7FFFFFFFull || cols > 0x7FFFFFFFull) fail(Errc::TooLarge, "image too large");
  if (row_base + out_rows > rows || in_row0 > (row_base > 0 ? row_base - 1 : 0))
    fail(Errc::BadValue, "band outside the image or missing its halo row");
  if (out_rows == 0) return;
  // phase: 0 RGGB (0,0), 1 BGGR (1,1), 2 GRBG (0,1), 3 GBRG (1,0)
  static const int kDr[4] = {0, 1, 0, 1}, kDc[4] = {0, 1, 1, 0};
  const int dr = kDr[phase & 3], dc = kDc[phase & 3];
  const std::uint64_t plane = out_rows * cols;
  // 128-bit paths need every row and every plane to start 16-byte aligned.
  const int vec_ok = (cols % 8 == 0) && (plane % 8 == 0) &&
                     (((reinterpret_cast<std::uintptr_t>(out) | reinterpret_cast<std::uintptr_t>(in)) & 15) == 0);
  // The column phase selects the kernel (site types are compile-time per
  // column).  Rows per thread: 4 for bilinear, 8 for gradient (16384^2 on a
  // B200: bilinear 0.340 / 0.346 ms, gradient 0.383 / 0.368 ms at 4 / 8);
  // GPCX_DEMOSAIC_RPT=4|8 overrides for A/B runs.
  static const int rpt_env = [] {
    const char* v = std::getenv("GPCX_DEMOSAIC_RPT");
    return v == nullptr ? 0 : (v[0] == '8' ? 8 : 4);
  }();
  const int rpt = rpt_env != 0 ? rpt_env : (gradient ? 8 : 4);
  const std::uint64_t tr = 8u * rpt;
  const dim3 grid(static_cast<unsigned>((cols + TC - 1) / TC),
                  static_cast<unsigned>((out_rows + tr - 1) / tr));
  if (grid.y > 65535) fail(Errc::TooLarge, "too many rows for the tile grid");
  const bool band = row_base != 0 || in_row0 != 0 || out_rows != rows;
  auto pick = [&](auto whole, auto banded) { return band ? banded : whole; };
  auto kernel =
      rpt == 8
          ? (gradient ? (dc ? pick(demosaic_kernel<true, 1, 8, false>, demosaic_kernel<true, 1, 8, true>)
                            : pick(demosaic_kernel<true, 0, 8, false>, demosaic_kernel<true, 0, 8, true>))
                      : (dc ? pick(demosaic_kernel<false, 1, 8, false>, demosaic_kernel<false, 1, 8, true>)
                            : pick(demosaic_kernel<false, 0, 8, false>, demosaic_kernel<false, 0, 8, true>)))
          : (gradient ? (dc ? pick(demosaic_kernel<true, 1, 4, false>, demosaic_kernel<true, 1, 4, true>)
                            : pick(demosaic_kernel<true, 0, 4, false>, demosaic_kernel<true, 0, 4, true>))
                      : (dc ? pick(demosaic_kernel<false, 1, 4, false>, demosaic_kernel<false, 1, 4, true>)
                            : pick(demosaic_kernel<false, 0, 4, false>, demosaic_kernel<false, 0, 4, true>)));
  kernel<<<grid, THREADS, 0, stream>>>(in, out, (int)rows, (int)cols, dr, vec_ok, (int)row_base,
                                       (int)in_row0, (int)out_rows);
  GPCX_LAUNCH_CHECK();
}

void launch(bool gradient, int phase, const std::uint16_t* in, std::uint16_t* out,
            std::uint64_t rows, std::uint64_t cols, cudaStream_t stream) {
  launch_band(gradient, phase, in, out, rows, cols, 0, 0, rows, stream);
}

}  // namespace gpcx::demosaic
