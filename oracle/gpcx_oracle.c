/*
 * gpcx_oracle.c -- CPU restatement of the LUT / MATMUL task path.
 * TEST INFRASTRUCTURE ONLY: see the header comment in gpcx_oracle.h for the
 * parity status ("unpinned by the reference", pinned by KATs + an
 * independent numpy restatement) and for who may call this.
 *
 * Parallel loops follow the reference substrate gpc::par::parallel_for
 * (proj/include/gpc/parexec.hpp:59-75: OpenMP static schedule over rows,
 * each body writing disjoint slots), so every result here is bitwise
 * independent of the thread count -- the same invariance contract the
 * reference states in proj/README.md:139-144.
 */
#include "gpcx_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

static int nthreads(int threads) {
  return threads > 0 ? threads : omp_get_max_threads();
}

int orc_max_threads(void) { return omp_get_max_threads(); }

uint64_t orc_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t orc_seed_b(uint64_t seed) { return orc_splitmix64(seed); }

/* SURVEY §8d "ramp12": 12-bit-like diagonal ramp plus +-32 noise. */
static uint16_t ramp12(uint64_t seed, uint64_t rows, uint64_t cols, uint64_t r,
                       uint64_t c) {
  const uint64_t h = orc_splitmix64(seed ^ (r * cols + c));
  const uint64_t span = (rows + cols >= 3) ? rows + cols - 2 : 1;
  int64_t v = 1024 + (int64_t)((3071ull * (r + c)) / span) +
              ((int64_t)(h >> 58) - 32);
  if (v < 0) v = 0;
  if (v > 65535) v = 65535;
  return (uint16_t)v;
}

void orc_synth_image(int kind, uint64_t seed, uint64_t rows, uint64_t cols,
                     uint64_t row0, uint64_t nrows, uint16_t* out) {
  const int64_t nr = (int64_t)nrows;
#pragma omp parallel for schedule(static)
  for (int64_t rr = 0; rr < nr; ++rr) {
    const uint64_t r = row0 + (uint64_t)rr;
    uint16_t* dst = out + (uint64_t)rr * cols;
    for (uint64_t c = 0; c < cols; ++c) {
      if (kind == ORC_IMG_RAMP12)
        dst[c] = ramp12(seed, rows, cols, r, c);
      else
        dst[c] = (uint16_t)(orc_splitmix64(seed ^ (r * cols + c)) & 0xFFFF);
    }
  }
}

static float mat_value(int kind, uint64_t h) {
  if (kind == ORC_MAT_EXACT8)
    return (float)(int8_t)(uint8_t)(h >> 56) * (1.0f / 128.0f);
  /* uniform32: 24-bit value in [-1, 1) */
  return (float)((double)(h >> 40) * (1.0 / 16777216.0) * 2.0 - 1.0);
}

void orc_synth_matrix(int kind, uint64_t seed, uint64_t rows, uint64_t cols,
                      uint64_t row0, uint64_t nrows, float* out) {
  (void)rows;
  const int64_t nr = (int64_t)nrows;
#pragma omp parallel for schedule(static)
  for (int64_t rr = 0; rr < nr; ++rr) {
    const uint64_t r = row0 + (uint64_t)rr;
    float* dst = out + (uint64_t)rr * cols;
    for (uint64_t c = 0; c < cols; ++c)
      dst[c] = mat_value(kind, orc_splitmix64(seed ^ (r * cols + c)));
  }
}

void orc_lut_hist(const uint16_t* img, uint64_t n, uint64_t* hist,
                  int threads) {
  const int t = nthreads(threads);
  uint32_t* part = (uint32_t*)calloc((size_t)t * 65536, sizeof(uint32_t));
  memset(hist, 0, 65536 * sizeof(uint64_t));
  const int64_t nn = (int64_t)n;
#pragma omp parallel num_threads(t)
  {
    uint32_t* h = part + (size_t)omp_get_thread_num() * 65536;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < nn; ++i) h[img[i]]++;
  }
  /* Combine in ascending thread order (integer sums: order-free anyway). */
  for (int w = 0; w < t; ++w) {
    const uint32_t* h = part + (size_t)w * 65536;
    for (int v = 0; v < 65536; ++v) hist[v] += h[v];
  }
  free(part);
}

int orc_lut_from_hist(const uint64_t* hist, int mode, uint16_t* lut,
                      orc_lut_stats* stats) {
  uint64_t n = 0;
  int lo = -1, hi = -1;
  for (int v = 0; v < 65536; ++v) {
    if (hist[v] == 0) continue;
    if (lo < 0) lo = v;
    hi = v;
    n += hist[v];
  }
  if (n == 0) return -1;
  stats->n = n;
  stats->lo = (uint32_t)lo;
  stats->hi = (uint32_t)hi;
  stats->cdf_min = (mode == ORC_LUT_STRETCH) ? 0 : hist[lo]; /* equalize only */

  if (mode == ORC_LUT_STRETCH) {
    const uint64_t span = (uint64_t)(hi - lo);
    for (uint64_t v = 0; v < 65536; ++v) {
      if (span == 0) {
        lut[v] = (uint16_t)v;
      } else if (v <= (uint64_t)lo) {
        lut[v] = 0;
      } else if (v >= (uint64_t)hi) {
        lut[v] = 65535;
      } else {
        lut[v] = (uint16_t)(((v - (uint64_t)lo) * 65535u + span / 2) / span);
      }
    }
    return 0;
  }

  /* equalize */
  const uint64_t cdf_min = hist[lo];
  const uint64_t d = n - cdf_min;
  uint64_t cdf = 0;
  for (int v = 0; v < 65536; ++v) {
    cdf += hist[v];
    if (d == 0) {
      lut[v] = (uint16_t)v;
    } else if (v < lo) {
      lut[v] = 0;
    } else {
      lut[v] = (uint16_t)(((cdf - cdf_min) * 65535u + d / 2) / d);
    }
  }
  return 0;
}

int orc_lut_gen(const uint16_t* img, uint64_t n, int mode, uint16_t* lut,
                orc_lut_stats* stats, int threads) {
  uint64_t* hist = (uint64_t*)malloc(65536 * sizeof(uint64_t));
  orc_lut_hist(img, n, hist, threads);
  const int rc = orc_lut_from_hist(hist, mode, lut, stats);
  free(hist);
  return rc;
}

void orc_lut_apply(const uint16_t* lut, const uint16_t* in, uint16_t* out,
                   uint64_t n, int threads) {
  const int64_t nn = (int64_t)n;
#pragma omp parallel for num_threads(nthreads(threads)) schedule(static)
  for (int64_t i = 0; i < nn; ++i) out[i] = lut[in[i]];
}

int orc_lut_correct(const uint16_t* in, uint16_t* out, uint64_t n, int mode,
                    uint16_t* lut, orc_lut_stats* stats, int threads) {
  const int rc = orc_lut_gen(in, n, mode, lut, stats, threads);
  if (rc != 0) return rc;
  orc_lut_apply(lut, in, out, n, threads);
  return 0;
}

uint64_t orc_digest_u16(const uint16_t* v, uint64_t n, uint64_t index0) {
  uint64_t total = 0;
  const int64_t nn = (int64_t)n;
#pragma omp parallel for reduction(+ : total) schedule(static)
  for (int64_t i = 0; i < nn; ++i)
    total += orc_splitmix64(((index0 + (uint64_t)i) << 16) | v[i]);
  return total;
}

static uint32_t f2u(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  return u;
}
static float u2f(uint32_t u) {
  float x;
  memcpy(&x, &u, 4);
  return x;
}

float orc_round_tf32(float x) {
  uint32_t u = f2u(x);
  if ((u & 0x7F800000u) == 0x7F800000u) return x; /* inf / nan */
  u = (u + 0x1000u) & 0xFFFFE000u;                 /* ties away from zero */
  return u2f(u);
}

float orc_round_bf16(float x) {
  uint32_t u = f2u(x);
  if ((u & 0x7F800000u) == 0x7F800000u) {
    if (u & 0x007FFFFFu) return u2f((u | 0x00400000u) & 0xFFFF0000u);
    return x;
  }
  u += 0x7FFFu + ((u >> 16) & 1u); /* ties to even */
  return u2f(u & 0xFFFF0000u);
}

void orc_round_matrix(int prec, const float* in, float* out, uint64_t count,
                      int threads) {
  const int64_t nn = (int64_t)count;
#pragma omp parallel for num_threads(nthreads(threads)) schedule(static)
  for (int64_t i = 0; i < nn; ++i) {
    if (prec == ORC_PREC_TF32)
      out[i] = orc_round_tf32(in[i]);
    else if (prec == ORC_PREC_BF16)
      out[i] = orc_round_bf16(in[i]);
    else
      out[i] = in[i];
  }
}

void orc_matmul_f64(uint64_t m, uint64_t n, uint64_t k, const float* A,
                    const float* B, const uint64_t* rows, uint64_t nrows,
                    double* C, double* absprod, int threads) {
  (void)m;
  const int64_t nr = (int64_t)nrows;
#pragma omp parallel num_threads(nthreads(threads))
  {
    double* acc = (double*)malloc(n * sizeof(double));
    double* aacc = absprod ? (double*)malloc(n * sizeof(double)) : NULL;
#pragma omp for schedule(static)
    for (int64_t rr = 0; rr < nr; ++rr) {
      const uint64_t i = rows ? rows[rr] : (uint64_t)rr;
      memset(acc, 0, n * sizeof(double));
      if (aacc) memset(aacc, 0, n * sizeof(double));
      const float* arow = A + i * k;
      for (uint64_t kk = 0; kk < k; ++kk) {
        const double a = (double)arow[kk];
        const float* brow = B + kk * n;
        for (uint64_t j = 0; j < n; ++j) acc[j] += a * (double)brow[j];
        if (aacc) {
          const double aa = fabs(a);
          for (uint64_t j = 0; j < n; ++j) aacc[j] += aa * fabs((double)brow[j]);
        }
      }
      memcpy(C + (uint64_t)rr * n, acc, n * sizeof(double));
      if (aacc) memcpy(absprod + (uint64_t)rr * n, aacc, n * sizeof(double));
    }
    free(acc);
    free(aacc);
  }
}

void orc_matmul_f32(uint64_t m, uint64_t n, uint64_t k, const float* A,
                    const float* B, float* C, int threads) {
  /* Four C rows per pass so each streamed row of B is reused 4x. */
  const int64_t blocks = (int64_t)((m + 3) / 4);
#pragma omp parallel num_threads(nthreads(threads))
  {
    double* acc = (double*)malloc(4 * n * sizeof(double));
#pragma omp for schedule(static)
    for (int64_t b = 0; b < blocks; ++b) {
      const uint64_t i0 = (uint64_t)b * 4;
      const uint64_t ni = (m - i0) < 4 ? (m - i0) : 4;
      memset(acc, 0, 4 * n * sizeof(double));
      for (uint64_t kk = 0; kk < k; ++kk) {
        const float* brow = B + kk * n;
        for (uint64_t r = 0; r < ni; ++r) {
          const double a = (double)A[(i0 + r) * k + kk];
          double* ar = acc + r * n;
          for (uint64_t j = 0; j < n; ++j) ar[j] += a * (double)brow[j];
        }
      }
      for (uint64_t r = 0; r < ni; ++r)
        for (uint64_t j = 0; j < n; ++j)
          C[(i0 + r) * n + j] = (float)acc[r * n + j];
    }
    free(acc);
  }
}
