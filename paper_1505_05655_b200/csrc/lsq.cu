// lsq.cu -- LSQ_POLYFIT on the GPU (fourth "next" row),
// bit-identical to the reference's f64 normal-equation fit
// (proj/src/lsq.cpp:44-223, proj/include/gpc/lsq.hpp:14-28):
//
//   per scan line y[0..pixels), x = i, s = max(1, pixels-1), t_i = x_i / s
//   S_p = sum_i t_i^p (p <= 2m),  T_j = sum_i t_i^j * y_i (j <= m)
//   A[j][k] = S_{j+k}, solve A c' = T by Gaussian elimination with partial
//   pivoting (Singular below 1e-12 * max|A|), c_k = c'_k / s^k,
//   sse = sum_i (y_i - horner(c, x_i))^2.
//
// Bit identity needs the reference's exact operation order:
//   * every sum is gpc::par::reduce_sum (parexec.hpp:86-103): sequential
//     within fixed 4096-element chunks from 0.0, chunk partials combined in
//     ascending order from 0.0 -- here one thread per (line, chunk), then one
//     thread per line for the combine;
//   * t^p is ipow's repeated multiplication from 1.0 (lsq.cpp:15-19), which
//     the running product t^p = t^(p-1) * t reproduces exactly;
//   * no fused multiply-add anywhere: the reference is built for baseline
//     x86-64 (no FMA), so every product and sum here is an explicit
//     __dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn.
// The power sums S_p depend only on `pixels`, so they are computed once and
// shared by all lines (the reference recomputes identical values per line).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "cuda_util.hpp"
#include "kernels.hpp"

namespace gpcx::lsq {

namespace {

constexpr int kChunk = 4096;  // gpc::par::ExecPlan::kChunk
constexpr int kMaxM1 = kMaxOrder + 1;

__device__ __forceinline__ double sample(const void* y, int dtype_f32, std::uint64_t idx) {
  return dtype_f32 ? static_cast<double>(static_cast<const float*>(y)[idx])
                   : static_cast<const double*>(y)[idx];
}

// S partials: one thread per chunk of x = 0..pixels-1.
__global__ void power_partials(std::uint64_t pixels, double scale, int max_p, double* part) {
  const std::uint64_t c = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const std::uint64_t nchunks = (pixels + kChunk - 1) / kChunk;
  if (c >= nchunks) return;
  double acc[2 * kMaxOrder + 1];
  for (int p = 0; p <= max_p; ++p) acc[p] = 0.0;
  const std::uint64_t lo = c * kChunk, hi = min(pixels, lo + kChunk);
  for (std::uint64_t i = lo; i < hi; ++i) {
    const double t = __ddiv_rn(static_cast<double>(i), scale);
    double tp = 1.0;
    for (int p = 0; p <= max_p; ++p) {
      acc[p] = __dadd_rn(acc[p], tp);
      tp = __dmul_rn(tp, t);
    }
  }
  for (int p = 0; p <= max_p; ++p) part[c * (2 * kMaxOrder + 1) + p] = acc[p];
}

// T partials and the first non-finite sample: one thread per (line, chunk).
__global__ void moment_partials(const void* y, int dtype_f32, std::uint64_t lines,
                                std::uint64_t pixels, double scale, int m, double* part,
                                unsigned long long* first_bad) {
  const std::uint64_t nchunks = (pixels + kChunk - 1) / kChunk;
  const std::uint64_t g = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= lines * nchunks) return;
  const std::uint64_t line = g / nchunks, c = g % nchunks;
  double acc[kMaxM1];
  for (int j = 0; j <= m; ++j) acc[j] = 0.0;
  const std::uint64_t lo = c * kChunk, hi = min(pixels, lo + kChunk);
  unsigned long long bad = ~0ull;
  for (std::uint64_t i = lo; i < hi; ++i) {
    const double yi = sample(y, dtype_f32, line * pixels + i);
    if (!isfinite(yi) && bad == ~0ull) bad = i;
    const double t = __ddiv_rn(static_cast<double>(i), scale);
    double tp = 1.0;
    for (int j = 0; j <= m; ++j) {
      acc[j] = __dadd_rn(acc[j], __dmul_rn(tp, yi));
      tp = __dmul_rn(tp, t);
    }
  }
  for (int j = 0; j <= m; ++j) part[g * kMaxM1 + j] = acc[j];
  if (bad != ~0ull) atomicMin(&first_bad[line], bad);
}

// Per line: combine partials in ascending chunk order, solve, unscale.
// status[line] = {code, col, best, floor} for the host to word the error.
__global__ void solve_lines(const double* spart, const double* tpart, std::uint64_t lines,
                            std::uint64_t pixels, double scale, int m,
                            const unsigned long long* first_bad, double* coeffs,
                            double* status) {
  const std::uint64_t line = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (line >= lines) return;
  const std::uint64_t nchunks = (pixels + kChunk - 1) / kChunk;
  const int n = m + 1;
  double* st = status + line * 4;
  st[0] = 0.0;
  if (first_bad[line] != ~0ull) {
    st[0] = 1.0;  // non-finite sample
    st[1] = static_cast<double>(first_bad[line]);
    return;
  }
  if (pixels < static_cast<std::uint64_t>(n)) {
    st[0] = 2.0;  // insufficient points
    return;
  }
  double S[2 * kMaxOrder + 1], T[kMaxM1];
  for (int p = 0; p <= 2 * m; ++p) {
    double tot = 0.0;
    for (std::uint64_t c = 0; c < nchunks; ++c)
      tot = __dadd_rn(tot, spart[c * (2 * kMaxOrder + 1) + p]);
    S[p] = tot;
  }
  for (int j = 0; j <= m; ++j) {
    double tot = 0.0;
    for (std::uint64_t c = 0; c < nchunks; ++c)
      tot = __dadd_rn(tot, tpart[(line * nchunks + c) * kMaxM1 + j]);
    T[j] = tot;
  }
  double a[kMaxM1][kMaxM1], b[kMaxM1];
  double max_abs = 0.0;
  for (int j = 0; j < n; ++j) {
    b[j] = T[j];
    for (int k = 0; k < n; ++k) {
      a[j][k] = S[j + k];
      max_abs = fmax(max_abs, fabs(a[j][k]));
    }
  }
  const double pivot_floor = __dmul_rn(1e-12, max_abs);
  for (int col = 0; col < n; ++col) {
    int pivot = col;
    double best = fabs(a[col][col]);
    for (int r = col + 1; r < n; ++r) {
      const double mag = fabs(a[r][col]);
      if (mag > best) {
        best = mag;
        pivot = r;
      }
    }
    if (best == 0.0 || best < pivot_floor) {
      st[0] = 3.0;  // singular
      st[1] = col;
      st[2] = best;
      st[3] = pivot_floor;
      return;
    }
    if (pivot != col) {
      for (int k = 0; k < n; ++k) {
        const double tmp = a[col][k];
        a[col][k] = a[pivot][k];
        a[pivot][k] = tmp;
      }
      const double tb = b[col];
      b[col] = b[pivot];
      b[pivot] = tb;
    }
    for (int r = col + 1; r < n; ++r) {
      const double f = __ddiv_rn(a[r][col], a[col][col]);
      if (f == 0.0) continue;
      a[r][col] = 0.0;
      for (int k = col + 1; k < n; ++k) a[r][k] = __dsub_rn(a[r][k], __dmul_rn(f, a[col][k]));
      b[r] = __dsub_rn(b[r], __dmul_rn(f, b[col]));
    }
  }
  double x[kMaxM1];
  for (int r = n - 1; r >= 0; --r) {
    double acc = b[r];
    for (int k = r + 1; k < n; ++k) acc = __dsub_rn(acc, __dmul_rn(a[r][k], x[k]));
    x[r] = __ddiv_rn(acc, a[r][r]);
  }
  for (int k = 0; k < n; ++k) {
    double sk = 1.0;
    for (int i = 0; i < k; ++i) sk = __dmul_rn(sk, scale);
    coeffs[line * (kMaxM1 + 1) + k] = __ddiv_rn(x[k], sk);
  }
}

// SSE partials: one thread per (line, chunk); Horner without FMA.
__global__ void sse_partials(const void* y, int dtype_f32, std::uint64_t lines,
                             std::uint64_t pixels, int m, const double* coeffs,
                             const double* status, double* part) {
  const std::uint64_t nchunks = (pixels + kChunk - 1) / kChunk;
  const std::uint64_t g = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= lines * nchunks) return;
  const std::uint64_t line = g / nchunks, c = g % nchunks;
  if (status[line * 4] != 0.0) return;
  double cf[kMaxM1];
  for (int k = 0; k <= m; ++k) cf[k] = coeffs[line * (kMaxM1 + 1) + k];
  const std::uint64_t lo = c * kChunk, hi = min(pixels, lo + kChunk);
  double acc = 0.0;
  for (std::uint64_t i = lo; i < hi; ++i) {
    const double xi = static_cast<double>(i);
    double v = 0.0;
    for (int k = m; k >= 0; --k) v = __dadd_rn(__dmul_rn(v, xi), cf[k]);
    const double d = __dsub_rn(sample(y, dtype_f32, line * pixels + i), v);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  part[g] = acc;
}

__global__ void sse_combine(const double* part, std::uint64_t lines, std::uint64_t pixels, int m,
                            const double* status, double* coeffs) {
  const std::uint64_t line = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (line >= lines || status[line * 4] != 0.0) return;
  const std::uint64_t nchunks = (pixels + kChunk - 1) / kChunk;
  double tot = 0.0;
  for (std::uint64_t c = 0; c < nchunks; ++c) tot = __dadd_rn(tot, part[line * nchunks + c]);
  coeffs[line * (kMaxM1 + 1) + (m + 1)] = tot;  // sse after the coefficients
}

unsigned blocks(std::uint64_t n, unsigned t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

std::uint64_t workspace_bytes(std::uint64_t lines, std::uint64_t pixels) {
  const std::uint64_t nchunks = (pixels + kChunk - 1) / kChunk;
  return 8 * (nchunks * (2 * kMaxOrder + 1) + lines * nchunks * kMaxM1 + lines * nchunks +
              lines * (kMaxM1 + 1) + lines * 4 + lines) + 256;
}

void launch(const void* y, bool dtype_f32, std::uint64_t lines, std::uint64_t pixels, int order,
            double* out_coeffs, double* out_status, void* ws, cudaStream_t stream) {
  const std::uint64_t nchunks = (pixels + kChunk - 1) / kChunk;
  const double scale = pixels - 1 > 1 ? static_cast<double>(pixels - 1) : 1.0;
  auto* base = static_cast<double*>(ws);
  double* spart = base;
  double* tpart = spart + nchunks * (2 * kMaxOrder + 1);
  double* epart = tpart + lines * nchunks * kMaxM1;
  auto* bad = reinterpret_cast<unsigned long long*>(epart + lines * nchunks);
  GPCX_CUDA(cudaMemsetAsync(bad, 0xFF, lines * sizeof(unsigned long long), stream));
  power_partials<<<blocks(nchunks, 128), 128, 0, stream>>>(pixels, scale, 2 * order, spart);
  GPCX_LAUNCH_CHECK();
  moment_partials<<<blocks(lines * nchunks, 128), 128, 0, stream>>>(
      y, dtype_f32, lines, pixels, scale, order, tpart, bad);
  GPCX_LAUNCH_CHECK();
  solve_lines<<<blocks(lines, 64), 64, 0, stream>>>(spart, tpart, lines, pixels, scale, order, bad,
                                                     out_coeffs, out_status);
  GPCX_LAUNCH_CHECK();
  sse_partials<<<blocks(lines * nchunks, 128), 128, 0, stream>>>(y, dtype_f32, lines, pixels, order,
                                                                  out_coeffs, out_status, epart);
  GPCX_LAUNCH_CHECK();
  sse_combine<<<blocks(lines, 64), 64, 0, stream>>>(epart, lines, pixels, order, out_status,
                                                     out_coeffs);
  GPCX_LAUNCH_CHECK();
}

}  // namespace gpcx::lsq
