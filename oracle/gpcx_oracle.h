/*
 * gpcx_oracle.h -- CPU restatement of the LUT / MATMUL task path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (libgpcx.so, the
 * executor, the kernels) links, calls or executes this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * use it, and there only as the checker / the CPU baseline.
 *
 * Parity status: the reference (/root/reference, `gpc`) implements no LUT
 * generation, LUT apply or matrix multiply -- PAPER.md:32 names them only as
 * motivating examples, and SURVEY.md §0.3 / §8c record that no reference
 * test, golden vector or fixture pins their arithmetic.  This oracle is
 * therefore a RESTATEMENT of the task contract written down in SURVEY.md
 * §8a' (formulas) and §8d (synthetic inputs, tolerances), following the
 * reference's conventions:
 *   - u16 little-endian row-major payloads   (proj/src/demosaic.cpp:177-209)
 *   - integer round-half-up "(sum + n/2)/n"  (proj/src/demosaic.cpp:37-46)
 *   - row-parallel, worker-count-invariant   (proj/include/gpc/parexec.hpp:11-31,59-75)
 *   - row-major f64-accumulating matrices    (proj/include/gpc/lsq.hpp:34-43)
 *   - independent serial oracle style        (proj/reference/reference.cpp:58-117)
 * Arithmetic parity is "unpinned by the reference"; it is pinned instead by
 * hand-computed known-answer tests (tests/test_oracle.py, SURVEY §8c list)
 * and by a second, independent numpy restatement (tests/oracle_np.py) that
 * must agree bit-for-bit.  The wire / dispatch behaviour IS pinned against
 * the reference itself, compiled from its own sources into oracle/_ref/.
 */
#ifndef GPCX_ORACLE_H
#define GPCX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_LUT_EQUALIZE = 0, ORC_LUT_STRETCH = 1 };
enum { ORC_IMG_RAMP12 = 0, ORC_IMG_UNIFORM16 = 1 };
enum { ORC_MAT_EXACT8 = 0, ORC_MAT_UNIFORM32 = 1 };
enum { ORC_PREC_F32 = 0, ORC_PREC_TF32 = 1, ORC_PREC_BF16 = 2 };

typedef struct orc_lut_stats {
  uint64_t n;        /* pixels */
  uint32_t lo, hi;   /* min / max sample */
  uint64_t cdf_min;  /* equalize: cdf at the smallest present value */
} orc_lut_stats;

/* Counter-based generator.  Same bits on CPU and GPU. */
uint64_t orc_splitmix64(uint64_t x);

/* Rows [row0, row0+nrows) of a rows x cols synthetic image. */
void orc_synth_image(int kind, uint64_t seed, uint64_t rows, uint64_t cols,
                     uint64_t row0, uint64_t nrows, uint16_t* out);
/* Rows [row0, row0+nrows) of a rows x cols synthetic f32 matrix. */
void orc_synth_matrix(int kind, uint64_t seed, uint64_t rows, uint64_t cols,
                      uint64_t row0, uint64_t nrows, float* out);
/* Seed of matrix B derived from the request seed (A uses the seed itself). */
uint64_t orc_seed_b(uint64_t seed);

/* 65536-bin histogram, u64 counts. */
void orc_lut_hist(const uint16_t* img, uint64_t n, uint64_t* hist, int threads);
/* LUT from a histogram (SURVEY §8a' formulas).  Returns 0, or -1 if n == 0. */
int orc_lut_from_hist(const uint64_t* hist, int mode, uint16_t* lut,
                      orc_lut_stats* stats);
int orc_lut_gen(const uint16_t* img, uint64_t n, int mode, uint16_t* lut,
                orc_lut_stats* stats, int threads);
void orc_lut_apply(const uint16_t* lut, const uint16_t* in, uint16_t* out,
                   uint64_t n, int threads);
int orc_lut_correct(const uint16_t* in, uint16_t* out, uint64_t n, int mode,
                    uint16_t* lut, orc_lut_stats* stats, int threads);

/* Position-keyed, order-independent digest of a u16 array whose first
 * element has global index index0:  sum_i splitmix64((i << 16) | v_i). */
uint64_t orc_digest_u16(const uint16_t* v, uint64_t n, uint64_t index0);

/* Input rounding the tensor-core paths apply (so the f64 oracle can be run
 * on exactly the operands the hardware sees). */
float orc_round_tf32(float x);  /* round-to-nearest, ties away (cvt.rna.tf32.f32) */
float orc_round_bf16(float x);  /* round-to-nearest-even (cvt.rn.bf16.f32) */
void orc_round_matrix(int prec, const float* in, float* out, uint64_t count,
                      int threads);

/* C[i,:] = sum_k A[i,k] * B[k,:] accumulated in f64, for the rows listed in
 * `rows` (or all m rows when rows == NULL; then nrows must equal m).
 * Also returns sum_k |A[i,k]|*|B[k,j]| in `absprod` when non-NULL (the
 * tolerance scale of SURVEY §8d).  Row-major everywhere; C/absprod are
 * nrows x n. */
void orc_matmul_f64(uint64_t m, uint64_t n, uint64_t k, const float* A,
                    const float* B, const uint64_t* rows, uint64_t nrows,
                    double* C, double* absprod, int threads);

/* CPU-baseline matmul producing f32 output (f64 accumulate, then rounded). */
void orc_matmul_f32(uint64_t m, uint64_t n, uint64_t k, const float* A,
                    const float* B, float* C, int threads);

int orc_max_threads(void);

#ifdef __cplusplus
}
#endif

#endif
