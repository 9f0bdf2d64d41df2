// lut.cu -- LUT generation and LUT-apply image correction for sm_100a.
//
// Task contract: SURVEY.md §8a' (LUT_GEN / LUT_APPLY / LUT_CORRECT), u16 LE
// row-major samples as in the reference codec (proj/src/demosaic.cpp:177-209),
// integer round-half-up as in proj/src/demosaic.cpp:37-46.  Results are
// bit-identical to oracle/gpcx_oracle.c and independent of the CTA count /
// GPU count (the parexec invariance contract, proj/include/gpc/parexec.hpp:11-31).
//
// Kernels (see DESIGN.md for the roofline of each):
//   fused_kernel    the equalize path, one cooperative launch, phases
//                   selected per call: histogram (1 CTA/SM, 128 KiB smem of
//                   packed u16 pairs + a 64 KiB u32 window for narrow data,
//                   128-bit streaming loads, 2 B/px; from 2^25 samples it
//                   also writes the 1 B/px residual plane) -> partial merge
//                   -> LUT -> apply (4 B/px, or 1 + 2 B/px from the plane).
//   stretch_fused_kernel  LUT_CORRECT stretch, one cooperative launch:
//                   min/max (2 B/px) -> grid sync -> per-CTA LUT in smem ->
//                   apply (4 B/px).
//   minmax_kernel   warp-shuffle (redux) min/max for LUT_GEN stretch and
//                   non-co-aligned LUT_CORRECT stretch.  2 B/px read.
//   from_minmax     stretch LUT.
//   apply_kernel    LUT_APPLY: persistent, LUT staged in 128 KiB smem,
//                   128-bit loads/stores, 8 gathers per vector.   4 B/px.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "cuda_util.hpp"
#include "kernels.hpp"

namespace gpcx {

int device_sm_count() {
  static thread_local int cached_dev = -1;
  static thread_local int cached_sms = 0;
  int dev = 0;
  GPCX_CUDA(cudaGetDevice(&dev));
  if (dev != cached_dev) {
    GPCX_CUDA(cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount,
                                     dev));
    cached_dev = dev;
  }
  return cached_sms;
}

namespace lut {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 1024;
constexpr std::uint64_t kOverflowOff = 0;
constexpr std::uint64_t kHistOff = 256 * 1024;
constexpr std::uint64_t kMinMaxOff = 512 * 1024;
constexpr std::uint64_t kBlocksOff = kMinMaxOff + 4 * 1024;  // 128 slice summaries (2 KiB)
constexpr std::uint64_t kPartsOff = kMinMaxOff + 8 * 1024;
constexpr int kSmemHist = kWords * 4 + 65536;  // 128 KiB packed bins + the 64 KiB u32 window
constexpr int kSmemLut = kBins * 2;    // 128 KiB
constexpr int kUnroll = 4;

// u32 work counters of the apply pass's dynamic tail (apply_image) and of
// the coded count pass's (count_tail_coded, the next word), in the unused
// end of the min/max slot area; the apply's is reset before the grid sync
// that precedes every cooperative apply, the count's after the grid sync
// that ends the count pass (so it is zero at the next launch).
constexpr std::uint64_t kTailOff = kMinMaxOff + 4 * 1024 - 64;
static_assert(kMaxParts * 8 <= 4 * 1024 - 64, "min/max slot area");

// Streaming image load.  Coherent (no .nc): the LUT kernels may write their
// output over their input (in == out) within the same launch, and PTX
// defines .nc loads only on memory that is read-only for the whole kernel.
// L1::no_allocate keeps the stream out of L1 like the .nc path did.
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Packed smem histogram: logical word w holds bin 2w in its low half and
// bin 2w+1 in its high half, so the word equals count(2w) +
// 65536*count(2w+1) mod 2^32.
//
// Bank layout.  Values with trailing zero bits -- MSB-aligned 8 / 10 / 12
// bit sensor data, multiples of 2^k -- put every lane of a warp on the same
// bank (8-bit data x 128: 7.4 ms instead of 1.2 at 32768^2).  Such images
// use a swizzled layout: word w at physical word swz1(w) / swz2(w), which
// XOR bits 5-9 (and 10-14) into the bank bits 0-4 (bijections that only
// permute the words of each 32-word group, each its own inverse).  The LUT staged in
// smem for the apply pass uses the same layout.  The choice is made per
// launch from a fixed sample of the image (`sample_layout`); it changes
// only where counts live, never their values.
// Two strengths, picked from the sample's trailing zero count tz: tz 3-6
// (12 / 10-bit data) XOR only bits 5-9 -- one instruction less per sample;
// tz >= 7 (8-bit data) needs bits 10-14 as well (with bits 5-9 alone,
// multiples of 256 still land on 8 banks: 1.82 vs 1.40 ms at 32768^2).
__device__ __host__ __forceinline__ uint32_t swz1(uint32_t w) { return w ^ ((w >> 5) & 31u); }
__device__ __host__ __forceinline__ uint32_t swz2(uint32_t w) {
  return w ^ (((w >> 5) ^ (w >> 10)) & 31u);
}
// physical word of logical word w in layout kSwz (0 plain, 1, 2)
template <int kSwz>
__device__ __forceinline__ uint32_t phys_word(uint32_t w) {
  if constexpr (kSwz == 1) return swz1(w);
  else if constexpr (kSwz == 2) return swz2(w);
  else return w;
}
template <int kSwz>
__device__ __forceinline__ uint32_t word_of(uint32_t v) {
  return phys_word<kSwz>(v >> 1);
}

// Add k (<= 65535) samples of value v.  The thread whose atomic wraps a
// half sees it in the returned old value and books the lost 65536 (and,
// for a low-half carry into the high half, the spurious +1) into the global
// overflow counters; the merge adds them back mod 2^32.  Exact for any
// count < 2^32 and independent of the interleaving.
template <int kSwz>
__device__ __forceinline__ void count_k(uint32_t* bins, uint32_t* overflow, uint32_t v,
                                        uint32_t k) {
  const uint32_t hi_bin = v & 1u;
  const uint32_t old = atomicAdd(&bins[word_of<kSwz>(v)], hi_bin ? k << 16 : k);
  const uint32_t half = hi_bin ? old >> 16 : old & 0xFFFFu;
  if (half + k > 0xFFFFu) {
    atomicAdd(&overflow[v], 65536u);
    if (!hi_bin) {
      // carry into the high half: +1 there that is not a sample of v+1,
      // and possibly a wrap of the high half itself.
      atomicAdd(&overflow[v + 1], (old >> 16) == 0xFFFFu ? 65535u : 0xFFFFFFFFu);
    }
  }
}

template <int kSwz>
__device__ __forceinline__ void count_one(uint32_t* bins, uint32_t* overflow, uint32_t v) {
  const uint32_t hi_bin = v & 1u;
  const uint32_t inc = hi_bin ? 0x10000u : 1u;
  const uint32_t mask = hi_bin ? 0xFFFF0000u : 0x0000FFFFu;
  const uint32_t old = atomicAdd(&bins[word_of<kSwz>(v)], inc);
  if ((old & mask) == mask) {
    atomicAdd(&overflow[v], 65536u);
    if (!hi_bin)
      atomicAdd(&overflow[v + 1], (old >> 16) == 0xFFFFu ? 65535u : 0xFFFFFFFFu);
  }
}

// 8 samples per lane: the 8 returning atomics are issued back to back and
// their (rare) wrap checks OR-ed into one branch per vector instead of a
// branch (and its reconvergence pair) after each atomic -- C3 step 1.211 ->
// 1.195 ms.
template <int kSwz>
__device__ __forceinline__ void count_vec_plain(uint32_t* bins,
                                                uint32_t* overflow, uint4 q) {
  const uint32_t v[8] = {q.x & 0xFFFFu, q.x >> 16, q.y & 0xFFFFu, q.y >> 16,
                         q.z & 0xFFFFu, q.z >> 16, q.w & 0xFFFFu, q.w >> 16};
  uint32_t old[8];
  bool wrapped = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t hi_bin = v[j] & 1u;
    const uint32_t m = hi_bin ? 0xFFFF0000u : 0x0000FFFFu;
    old[j] = atomicAdd(&bins[word_of<kSwz>(v[j])], hi_bin ? 0x10000u : 1u);
    wrapped |= (old[j] & m) == m;
  }
  if (wrapped) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t hi_bin = v[j] & 1u;
      const uint32_t m = hi_bin ? 0xFFFF0000u : 0x0000FFFFu;
      if ((old[j] & m) != m) continue;
      atomicAdd(&overflow[v[j]], 65536u);
      if (!hi_bin)
        atomicAdd(&overflow[v[j] + 1], (old[j] >> 16) == 0xFFFFu ? 65535u : 0xFFFFFFFFu);
    }
  }
}

// Two vectors (16 samples) per lane: the 16 returning atomics back to back,
// then ONE conservative wrap test for all of them -- does any half of any
// returned word read 0xFFFF? (a SIMD u16x2 max over the 16 old values) --
// and the exact per-sample check only when it fires.  The exact per-sample
// test (mask select, and, compare: 3 instructions per sample) and its
// branch cost ~3% of the pass on the C3 scenes, whose random noise makes
// the atomics bank-conflict bound (count 493 -> 478 us), and ~30% where
// the samples of a warp fall on distinct banks and the pass becomes issue
// bound (profiles/r2/plane_trace.txt).  The test can fire spuriously (the
// other bin of a word at 0xFFFF); the slow path then finds nothing.
template <int kSwz>
__device__ __forceinline__ void count_pair_plain(uint32_t* bins, uint32_t* overflow, uint4 q0,
                                                 uint4 q1) {
  const uint32_t w[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
  uint32_t old[16];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t lo = w[j] & 0xFFFFu, hi = w[j] >> 16;
    old[2 * j] = atomicAdd(&bins[word_of<kSwz>(lo)], (lo & 1u) ? 0x10000u : 1u);
    old[2 * j + 1] = atomicAdd(&bins[word_of<kSwz>(hi)], (hi & 1u) ? 0x10000u : 1u);
  }
  uint32_t mx = __vmaxu2(__vmaxu2(old[0], old[1]), __vmaxu2(old[2], old[3]));
  mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(old[4], old[5]), __vmaxu2(old[6], old[7])));
  mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(old[8], old[9]), __vmaxu2(old[10], old[11])));
  mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(old[12], old[13]), __vmaxu2(old[14], old[15])));
  if ((mx & 0xFFFFu) != 0xFFFFu && mx < 0xFFFF0000u) return;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t v = (j & 1) ? w[j >> 1] >> 16 : w[j >> 1] & 0xFFFFu;
    const uint32_t hi_bin = v & 1u;
    const uint32_t m = hi_bin ? 0xFFFF0000u : 0x0000FFFFu;
    if ((old[j] & m) != m) continue;
    atomicAdd(&overflow[v], 65536u);
    if (!hi_bin)
      atomicAdd(&overflow[v + 1], (old[j] >> 16) == 0xFFFFu ? 65535u : 0xFFFFFFFFu);
  }
}

// Repetitive data (flat regions, binary or few-level images): on one word
// the lanes' returning atomics queue up, so a warp whose samples fall on
// few banks combines them first -- one or two atomics when the warp vector
// holds at most two values (flat / binary: warp min, max and a count),
// else one per distinct value per sample slot (__match_any_sync).
template <int kSwz>
__device__ __noinline__ void count_vec_few(uint32_t* bins, uint32_t* overflow, uint4 q,
                                           uint32_t mask) {
  const uint32_t v[8] = {q.x & 0xFFFFu, q.x >> 16, q.y & 0xFFFFu, q.y >> 16,
                         q.z & 0xFFFFu, q.z >> 16, q.w & 0xFFFFu, q.w >> 16};
  const uint32_t lane = threadIdx.x & 31u;
  const int leader = __ffs(mask) - 1;
  // flat warp vector: one atomic
  const uint32_t pair = v[0] | (v[0] << 16);
  const bool flat = (q.x == pair) & (q.y == pair) & (q.z == pair) & (q.w == pair);
  const uint32_t lead_v = __shfl_sync(mask, v[0], leader);  // every lane of mask
  if (__all_sync(mask, flat & (v[0] == lead_v))) {
    if (lane == static_cast<uint32_t>(leader)) count_k<kSwz>(bins, overflow, v[0], 8u * __popc(mask));
    return;
  }
  // at most two values (binary): the warp's min and max, and how many
  // samples equal the min -- two atomics in all
  uint32_t mn = v[0], mx = v[0];
#pragma unroll
  for (int j = 1; j < 8; ++j) {
    mn = min(mn, v[j]);
    mx = max(mx, v[j]);
  }
  mn = __reduce_min_sync(mask, mn);
  mx = __reduce_max_sync(mask, mx);
  bool two = true;
  uint32_t c_mn = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    two &= (v[j] == mn) | (v[j] == mx);
    c_mn += v[j] == mn;
  }
  if (__all_sync(mask, two)) {
    c_mn = __reduce_add_sync(mask, c_mn);
    if (lane == static_cast<uint32_t>(leader)) {
      const uint32_t total = 8u * __popc(mask);
      count_k<kSwz>(bins, overflow, mn, c_mn);
      if (c_mn < total) count_k<kSwz>(bins, overflow, mx, total - c_mn);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t peers = __match_any_sync(mask, v[j]);
    if (lane == static_cast<uint32_t>(__ffs(peers) - 1))
      count_k<kSwz>(bins, overflow, v[j], __popc(peers));
  }
}

// Few distinct words among the warp's first samples of the vectors?
template <int kSwz>
__device__ __forceinline__ uint32_t bank_bit(uint4 q) {
  return 1u << (word_of<kSwz>(q.x & 0xFFFFu) & 31u);
}

template <int kSwz>
__device__ __forceinline__ void count_vec(uint32_t* bins, uint32_t* overflow, uint4 q) {
  const uint32_t mask = __activemask();
  if (__popc(__reduce_or_sync(mask, bank_bit<kSwz>(q))) <= 4) count_vec_few<kSwz>(bins, overflow, q, mask);
  else count_vec_plain<kSwz>(bins, overflow, q);
}

// The main loop's two vectors share one probe (half its cost per sample).
template <int kSwz>
__device__ __forceinline__ void count_pair(uint32_t* bins, uint32_t* overflow, uint4 q0,
                                           uint4 q1) {
  const uint32_t mask = __activemask();
  if (__popc(__reduce_or_sync(mask, bank_bit<kSwz>(q0) | bank_bit<kSwz>(q1))) <= 6) {
    count_vec_few<kSwz>(bins, overflow, q0, mask);
    count_vec_few<kSwz>(bins, overflow, q1, mask);
  } else {
    count_pair_plain<kSwz>(bins, overflow, q0, q1);
  }
}

// ---- count policies: how one sample / vector / two vectors are counted --
constexpr uint32_t kWinBins = 16384;   // u32 window counters, 64 KiB of smem
constexpr uint32_t kNoWindow = 0xFFFFFFFFu;

template <int kSwz>
struct PlainCounter {  // packed u16 pairs, returning atomics, wrap test
  uint32_t* bins;
  uint32_t* overflow;
  __device__ __forceinline__ void one(uint32_t v) const { count_one<kSwz>(bins, overflow, v); }
  __device__ __forceinline__ void vec(uint4 q) const { count_vec_plain<kSwz>(bins, overflow, q); }
  __device__ __forceinline__ void pair(uint4 a, uint4 b) const {
    count_pair_plain<kSwz>(bins, overflow, a, b);
  }
};
template <int kSwz>
struct FewCounter {  // repetitive data too wide for the window: warp-combined counts
  uint32_t* bins;
  uint32_t* overflow;
  __device__ __forceinline__ void one(uint32_t v) const { count_one<kSwz>(bins, overflow, v); }
  __device__ __forceinline__ void vec(uint4 q) const { count_vec<kSwz>(bins, overflow, q); }
  __device__ __forceinline__ void pair(uint4 a, uint4 b) const {
    count_pair<kSwz>(bins, overflow, a, b);
  }
};
// Narrow data (the sampled values span < kWinBins - 2048): every value in
// [lo, lo + kWinBins) has its own u32 counter in a 64 KiB smem window,
// counted with red.shared (no return value, no wrap test: a CTA counts
// < 2^32 samples); the rest go to the packed histogram (plain layout).
// Packed pairs put neighbouring values -- a smooth image's warp samples --
// on the same word with different increments, which the atomic unit
// serialises: C3 ramp12's count 0.481 -> 0.390 ms in tools/hist_probe.cu
// (profiles/r2/hist_probe_window.txt); flat / few-level data in the window
// is fast too (many lanes' red on one counter run at the HBM rate).
// fold_window() moves the window into
// the packed histogram before the partial flush (the window's packed
// halves are untouched: every in-window sample went to the window).
template <int kSwz>
struct WindowCounter {
  uint32_t* bins;
  uint32_t* overflow;
  uint32_t* win;
  uint32_t lo;  // even; 0 when shifted
  uint32_t sh;  // 0, or the trailing zero bits of MSB-aligned data (lo 0)
  // per u16 half d = v - lo: in the window iff (d & reject) == 0
  __device__ __forceinline__ uint32_t reject() const { return sh == 0 ? 0xC000u : (1u << sh) - 1u; }
  __device__ __forceinline__ void one(uint32_t v) const {
    const uint32_t d = (v - lo) & 0xFFFFu;
    if (v >= lo && (d & reject()) == 0) atomicAdd(win + (d >> sh), 1u);
    else count_one<kSwz>(bins, overflow, v);
  }
  __device__ __forceinline__ void vec(uint4 q) const {
    one(q.x & 0xFFFFu); one(q.x >> 16); one(q.y & 0xFFFFu); one(q.y >> 16);
    one(q.z & 0xFFFFu); one(q.z >> 16); one(q.w & 0xFFFFu); one(q.w >> 16);
  }
  __device__ __forceinline__ void pair(uint4 a, uint4 b) const {
    // per u16 half v - lo (wrapping below lo: a narrow window's test bits
    // 14-15 catch it; a shifted window has lo 0)
    const uint32_t l2 = lo * 0x10001u;
    const uint32_t d[8] = {__vsub2(a.x, l2), __vsub2(a.y, l2), __vsub2(a.z, l2), __vsub2(a.w, l2),
                           __vsub2(b.x, l2), __vsub2(b.y, l2), __vsub2(b.z, l2), __vsub2(b.w, l2)};
    static_assert(kWinBins == 0x4000, "window test");
    const uint32_t any = d[0] | d[1] | d[2] | d[3] | d[4] | d[5] | d[6] | d[7];
    if (__all_sync(__activemask(), (any & (reject() * 0x10001u)) == 0)) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        atomicAdd(win + ((d[j] & 0xFFFFu) >> sh), 1u);
        atomicAdd(win + (d[j] >> (16 + sh)), 1u);
      }
    } else {
      vec(a);
      vec(b);
    }
  }
};

// Window counts into the packed histogram (all threads, after the count
// pass's barrier; a barrier must follow): counter i is value lo + (i << sh);
// its packed half gets the low 16 bits (the half was never touched: every
// sample of that value went to the window), the rest of a count above
// 65535 goes to the overflow counters the merge adds back.  Narrow window:
// counters 2i, 2i + 1 fill one word; shifted: one even value per word.
template <int kSwz>
__device__ __forceinline__ void fold_window(uint32_t* bins, uint32_t* overflow, const uint32_t* win,
                                            uint32_t lo, uint32_t sh) {
  if (sh == 0) {
    for (uint32_t i = threadIdx.x; i < kWinBins / 2; i += kThreads) {
      const uint2 c = reinterpret_cast<const uint2*>(win)[i];
      const uint32_t v0 = lo + 2 * i;
      bins[phys_word<kSwz>(v0 >> 1)] += (c.x & 0xFFFFu) | (c.y << 16);
      if (c.x > 0xFFFFu) atomicAdd(&overflow[v0], c.x & 0xFFFF0000u);
      if (c.y > 0xFFFFu) atomicAdd(&overflow[v0 + 1], c.y & 0xFFFF0000u);
    }
  } else {
    for (uint32_t i = threadIdx.x; i < kWinBins && (i << sh) <= 0xFFFFu; i += kThreads) {
      const uint32_t c = win[i];
      if (c == 0) continue;
      const uint32_t v = i << sh;  // even: the low half of its word
      bins[phys_word<kSwz>(v >> 1)] += c & 0xFFFFu;
      if (c > 0xFFFFu) atomicAdd(&overflow[v], c & 0xFFFF0000u);
    }
  }
}

// Per-launch choices from a fixed sample -- 256 pairs of adjacent samples
// spread over the image, the same in every CTA:
//   bits 0-1  smem layout: 0 plain; 1 / 2 swizzled when the OR of the
//          samples has 3-6 / >= 7 trailing zero bits (MSB-aligned data);
//   bit 2  repetitive data: >= 1/8 of the pairs are equal (flat regions,
//          binary or few-level images; noise-free ramps too) -> the count
//          pass probes each warp's diversity and combines equal values.
//          Ordinary images skip that probe (it costs ~2.5% on them).
//   bit 3  smooth data: >= 1/2 of the pairs differ by < 64 -> worth coding
//          the residual plane (fused_kernel); noise-like images skip its
//          per-block test, which would mark every block raw (~3% on them).
//          MSB-aligned data (>= 2 trailing zero bits) counts as smooth when
//          the pairs differ by < 64 steps of 2^tz; bits 8-11 then hold the
//          plane's residual shift min(tz, 8).
// and (`wlo`, `wsh`, optional) the count pass's u32 window (WindowCounter):
// either narrow data (plain layout, sampled values spanning less than
// kWinBins - 2048): first value `wlo` (even, the window centred on them),
// shift 0; or MSB-aligned data (>= 2 trailing zero bits): wlo 0 and shift
// = the trailing zeros, counter v >> shift for every v with those bits
// clear (all of [0, 65536)); else kNoWindow.
// Warp 0 computes the flags into *flags; the caller's next __syncthreads
// publishes them.  They change where and how counts are added, never what.
__device__ __forceinline__ void sample_layout(const std::uint16_t* img, std::uint64_t n,
                                              uint32_t* flags, uint32_t* wlo = nullptr,
                                              uint32_t* wsh = nullptr) {
  if (threadIdx.x >= 32) return;
  uint32_t o = 0, eq = 0, near = 0, mn = 0xFFFFu, mx = 0;
  uint32_t a[8] = {}, b[8] = {};
  if (n >= 2) {
    // 8 pairs per lane, all 16 loads in flight at once (this runs while
    // the other warps zero the histogram, and C1's whole kernel is ~40 us)
    const double step = static_cast<double>(n - 2) / 255.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const std::uint64_t p =
          static_cast<std::uint64_t>(static_cast<double>(threadIdx.x + 32 * k) * step);
      a[k] = __ldcg(img + p);
      b[k] = __ldcg(img + p + 1);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      o |= a[k] | b[k];
      eq += a[k] == b[k];
      near += (a[k] > b[k] ? a[k] - b[k] : b[k] - a[k]) < 64u;
      mn = min(mn, min(a[k], b[k]));
      mx = max(mx, max(a[k], b[k]));
    }
  } else if (n == 1 && threadIdx.x == 0) {
    o = img[0];
  }
  o = __reduce_or_sync(0xFFFFFFFFu, o);
  eq = __reduce_add_sync(0xFFFFFFFFu, eq);
  near = __reduce_add_sync(0xFFFFFFFFu, near);
  mn = __reduce_min_sync(0xFFFFFFFFu, mn);
  mx = __reduce_max_sync(0xFFFFFFFFu, mx);
  const uint32_t tz = o == 0 ? 32u : static_cast<uint32_t>(__ffs(o) - 1);
  // smooth in units of the data's step (MSB-aligned data: 2^tz)
  const uint32_t s8 = min(tz, 8u);
  uint32_t nearsh = 0;
  if (n >= 2) {
#pragma unroll
    for (int k = 0; k < 8; ++k) nearsh += ((a[k] > b[k] ? a[k] - b[k] : b[k] - a[k]) >> s8) < 64u;
  }
  nearsh = __reduce_add_sync(0xFFFFFFFFu, nearsh);
  if (threadIdx.x == 0) {
    const uint32_t layout = (n == 0 || tz < 3) ? 0u : (tz <= 6 ? 1u : 2u);
    // the residual plane: smooth data (raw units, or steps of 2^tz up to 2^8)
    uint32_t plane = 0;
    if (near >= 128) plane = 8u;
    else if (n >= 2 && tz >= 2 && tz < 32 && nearsh >= 128) plane = 8u | (s8 << 8);
    *flags = layout | (eq >= 32 ? 4u : 0u) | plane;
    if (wlo != nullptr) {
      uint32_t lo = kNoWindow, sh = 0;
      if (n >= 2 && tz >= 2 && tz < 32 && (tz >= 7 || nearsh >= 128)) {
        // MSB-aligned data, smooth or with few levels: counter v >> tz (random
        // data with 1024+ levels runs faster on the swizzled packed bins)
        lo = 0;
        sh = min(tz, 15u);
      } else if (n >= 2 && layout == 0 && mx >= mn && mx - mn <= kWinBins - 2048) {
        const uint32_t pad = (kWinBins - (mx - mn)) / 2;
        lo = mn > pad ? mn - pad : 0u;
        lo = min(lo, 65536u - kWinBins) & ~1u;
      }
      *wlo = lo;
      *wsh = sh;
    }
  }
}

// Samples before the first 16-byte boundary (pointers are at least 2-byte
// aligned), rounded to whole samples.
__device__ __host__ __forceinline__ std::uint64_t head_len(const void* p,
                                                           std::uint64_t n) {
  const std::uint64_t mis = reinterpret_cast<std::uintptr_t>(p) & 15u;
  const std::uint64_t h = ((16u - mis) & 15u) >> 1;
  return h < n ? h : n;
}

// LUT entry v of the smem LUT (u16 entries, two per word; swizzled words
// when kSwz -- see the bank layout note above).
template <int kSwz>
__device__ __forceinline__ uint32_t lut_at(const std::uint16_t* s_lut, uint32_t v) {
  return kSwz ? s_lut[(phys_word<kSwz>(v >> 1) << 1) | (v & 1u)] : s_lut[v];
}

template <int kSwz>
__device__ __forceinline__ uint4 lookup_vec(const std::uint16_t* s_lut, uint4 q) {
  uint4 r;
  r.x = lut_at<kSwz>(s_lut, q.x & 0xFFFFu) | (lut_at<kSwz>(s_lut, q.x >> 16) << 16);
  r.y = lut_at<kSwz>(s_lut, q.y & 0xFFFFu) | (lut_at<kSwz>(s_lut, q.y >> 16) << 16);
  r.z = lut_at<kSwz>(s_lut, q.z & 0xFFFFu) | (lut_at<kSwz>(s_lut, q.z >> 16) << 16);
  r.w = lut_at<kSwz>(s_lut, q.w & 0xFFFFu) | (lut_at<kSwz>(s_lut, q.w >> 16) << 16);
  return r;
}

// Stage the global LUT (logical order) into smem in the kSwz layout.
template <int kSwz>
__device__ __forceinline__ void stage_lut(uint4* smem, const std::uint16_t* lut_g) {
  if constexpr (kSwz) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(lut_g);
    uint32_t* dst = reinterpret_cast<uint32_t*>(smem);
    for (int w = threadIdx.x; w < kWords; w += blockDim.x) dst[phys_word<kSwz>(w)] = __ldcg(src + w);
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(lut_g);
    for (int i = threadIdx.x; i < kBins / 8; i += blockDim.x) smem[i] = __ldcg(src + i);
  }
}

// Histogram of img[0, n) into the packed smem bins; CTA `cta` of `ctas`
// (grid-stride over 128-bit vectors, two-vector software pipeline: the next
// stage's loads are in flight while this stage's 16 samples are counted).
template <class Ctr>
__device__ __forceinline__ void count_image(const std::uint16_t* img, std::uint64_t n, int cta,
                                            int ctas, const Ctr& ctr) {
  const std::uint64_t head = head_len(img, n);
  const std::uint64_t nvec = (n - head) >> 3;
  const std::uint64_t tail0 = head + (nvec << 3);
  if (cta == 0)
    for (std::uint64_t i = threadIdx.x; i < head; i += kThreads) ctr.one(img[i]);
  if (cta == ctas - 1)
    for (std::uint64_t i = tail0 + threadIdx.x; i < n; i += kThreads) ctr.one(img[i]);
  const uint4* body = reinterpret_cast<const uint4*>(img + head);
  const std::uint64_t stride = static_cast<std::uint64_t>(ctas) * kThreads;
  std::uint64_t i = static_cast<std::uint64_t>(cta) * kThreads + threadIdx.x;
  uint4 q[2], nq[2];
  bool have = i + stride < nvec;
  if (have) {
    q[0] = ld_stream(body + i);
    q[1] = ld_stream(body + i + stride);
  }
  while (have) {
    const std::uint64_t nx = i + 2 * stride;
    const bool nhave = nx + stride < nvec;
    if (nhave) {
      nq[0] = ld_stream(body + nx);
      nq[1] = ld_stream(body + nx + stride);
    }
    ctr.pair(q[0], q[1]);
    q[0] = nq[0];
    q[1] = nq[1];
    i = nx;
    have = nhave;
  }
  for (; i < nvec; i += stride) ctr.vec(ld_stream(body + i));
}

// out = LUT[in] over [0, n) with the LUT in smem; CTA `cta` of `ctas`.
// Two vectors per stage, the next stage's loads in flight while this one is
// looked up and stored (tools/apply_bench.cu: = cudaMemcpy D2D bandwidth).
// With `tail` (cooperative launches, counter zeroed before their last grid
// sync) the last 4 x ctas chunks of 8 vectors per thread are not assigned
// statically but taken chunk by chunk from the counter: CTAs do not stream
// at identical rates (the static split left a ~20 us spread between the
// first and the last CTA to finish, profiles/r1/fused_trace_v2_c3.txt), and
// the dynamic tail lets the early ones take the late ones' share.
template <int kSwz>
__device__ __forceinline__ void apply_image(const std::uint16_t* s_lut, const std::uint16_t* in,
                                            std::uint16_t* out, std::uint64_t n, int cta,
                                            int ctas, std::uint32_t* tail = nullptr) {
  constexpr std::uint64_t kChunk = 8ull * kThreads;  // vectors per tail chunk (128 KiB)
  const std::uint64_t tid = static_cast<std::uint64_t>(cta) * kThreads + threadIdx.x;
  const std::uint64_t stride = static_cast<std::uint64_t>(ctas) * kThreads;
  const std::uint64_t head = head_len(in, n);
  const std::uint64_t nvec = (n - head) >> 3;
  const std::uint64_t tail0 = head + (nvec << 3);
  if (tid < head) out[tid] = lut_at<kSwz>(s_lut, in[tid]);
  if (tid < n - tail0) out[tail0 + tid] = lut_at<kSwz>(s_lut, in[tail0 + tid]);
  const uint4* src = reinterpret_cast<const uint4*>(in + head);
  uint4* dst = reinterpret_cast<uint4*>(out + head);
  const std::uint64_t tail_chunks = 4ull * static_cast<std::uint64_t>(ctas);
  const bool dynamic = tail != nullptr && nvec >= 16 * tail_chunks * kChunk;
  const std::uint64_t static_end = dynamic ? nvec - tail_chunks * kChunk : nvec;
  constexpr int kU = 2;
  std::uint64_t i = tid;
  uint4 q[kU], nq[kU];
  bool have = i + (kU - 1) * stride < static_end;
  if (have) {
#pragma unroll
    for (int u = 0; u < kU; ++u) q[u] = ld_stream(src + i + u * stride);
  }
  while (have) {
    const std::uint64_t nx = i + kU * stride;
    const bool nhave = nx + (kU - 1) * stride < static_end;
    if (nhave) {
#pragma unroll
      for (int u = 0; u < kU; ++u) nq[u] = ld_stream(src + nx + u * stride);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) st_stream(dst + i + u * stride, lookup_vec<kSwz>(s_lut, q[u]));
#pragma unroll
    for (int u = 0; u < kU; ++u) q[u] = nq[u];
    i = nx;
    have = nhave;
  }
  for (; i < static_end; i += stride) st_stream(dst + i, lookup_vec<kSwz>(s_lut, ld_stream(src + i)));
  if (!dynamic) return;
  __shared__ std::uint32_t s_chunk;
  for (;;) {
    __syncthreads();  // the previous chunk index is consumed
    if (threadIdx.x == 0) s_chunk = atomicAdd(tail, 1u);
    __syncthreads();
    const std::uint64_t c = s_chunk;
    if (c >= tail_chunks) break;
    const std::uint64_t v0 = static_end + c * kChunk + threadIdx.x;
    uint4 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = ld_stream(src + v0 + u * kThreads);
#pragma unroll
    for (int u = 0; u < 8; ++u) st_stream(dst + v0 + u * kThreads, lookup_vec<kSwz>(s_lut, x[u]));
  }
}

// ---- the residual plane: a narrow copy of the image, count -> apply ------
// The packed-bin count pass is bound by the shared-memory atomic unit
// (~0.47 ms at C3 against a 0.335 ms read floor: HBM idles ~30% of it), the
// apply pass by HBM (2 B read + 2 B written per sample).  With room in the
// workspace (workspace_bytes(n)), the count pass also stores every
// 512-sample block (64 vectors: two adjacent 512-byte warp loads) whose
// samples lie in a 256-value window as a base word and one residual byte
// per sample (code_block); the apply pass reads that 1 B/px copy instead of
// the 2 B/px image.  Bytes move from the HBM-bound pass into the
// atomic-bound one: 2 + 1 (count) and 1 + 2 (apply) per sample instead of 2
// and 2 + 2 -- the same 6 B/px, but no pass idles HBM.  Other blocks
// (noise-like data) get base word kRawBlock and are applied from the image.
// MSB-aligned smooth data (sample_layout's shift sh = min(tz, 8)) is coded
// in steps of 2^sh: window [base, base + 256 << sh), residual
// (v - base) >> sh.  Exact by construction: v = base + (residual << sh).
// Block b = vectors [64b, 64b + 64) of the 16-byte-aligned body, lane l
// holding vectors 64b + l and 64b + 32 + l (residuals: 16 bytes at plane
// vector 32b + l); plane layout: u32 base[n >> 9] (256-byte rounded) | 512
// bytes per block.
constexpr uint32_t kRawBlock = 0x10000u;
constexpr std::uint64_t kPlaneMin = 1ull << 25;  // samples; below it the image stays in L2

__host__ __device__ __forceinline__ std::uint64_t plane_base_bytes(std::uint64_t n) {
  return ((n >> 9) * 4 + 255) & ~std::uint64_t{255};
}

// One block (the warp's 64 vectors, all lanes active).  Base = lane 0's
// first sample - (128 << sh) (clamped to [0, 65536 - (256 << sh)]); the
// block is narrow when every sample lies on the 2^sh grid in
// [base, base + (256 << sh)) -- tested on the plain 32-bit differences
// q - base (per u16 half): a half outside the window or off the grid
// leaves a bit outside [sh, sh + 8) set in its half (an underflowing low
// half included, given the clamp), and with none outside there is no
// borrow, so bits [sh, sh + 8) of each half are the residuals.  One
// shuffle and one vote per block, no min/max tree (a redux min/max version
// cost the then issue-sensitive count pass ~75 us at C3).
__device__ __forceinline__ void code_block(uint4 q0, uint4 q1, std::uint64_t blk, uint32_t lane,
                                           uint32_t* pbase, uint4* pres, uint32_t sh) {
  // sh > 0 (MSB-aligned data, steps of 2^sh): window [base, base + 256 << sh),
  // residual (v - base) >> sh; a sample off the step grid rejects the block
  const uint32_t f = __shfl_sync(0xFFFFFFFFu, q0.x, 0) & 0xFFFFu;
  const uint32_t half = 128u << sh, lim = 65536u - (256u << sh);
  const uint32_t base = min(max(f, half) - half, lim);
  const uint32_t b2 = base * 0x10001u;
  const uint4 d0 = make_uint4(q0.x - b2, q0.y - b2, q0.z - b2, q0.w - b2);
  const uint4 d1 = make_uint4(q1.x - b2, q1.y - b2, q1.z - b2, q1.w - b2);
  const uint32_t any = d0.x | d0.y | d0.z | d0.w | d1.x | d1.y | d1.z | d1.w;
  const uint32_t rej = (0xFFFFu & ~(0xFFu << sh)) * 0x10001u;
  const bool narrow = __all_sync(0xFFFFFFFFu, (any & rej) == 0);
  if (narrow) {
    auto r = [sh](uint32_t d) { return (d >> sh) & 0x00FF00FFu; };
    st_stream(pres + blk * 32 + lane,
              make_uint4(__byte_perm(r(d0.x), r(d0.y), 0x6420), __byte_perm(r(d0.z), r(d0.w), 0x6420),
                         __byte_perm(r(d1.x), r(d1.y), 0x6420), __byte_perm(r(d1.z), r(d1.w), 0x6420)));
  }
  if (lane == 0) pbase[blk] = narrow ? base : kRawBlock;
}

// The coded count pass's last blocks, 8-block chunks taken warp by warp
// from a counter (the next chunk's index requested while this one is
// counted).  Out of line so its registers do not crowd the main loop.
template <class Ctr>
__device__ __noinline__ void count_tail_coded(const uint4* body, std::uint64_t static_end,
                                              std::uint32_t tail_chunks, std::uint32_t* ctail,
                                              Ctr ctr, uint32_t* pbase, uint4* pres, uint32_t sh) {
  constexpr std::uint64_t kWChunk = 8;
  const uint32_t lane = threadIdx.x & 31u;
  std::uint32_t c = 0;
  if (lane == 0) c = atomicAdd(ctail, 1u);
  c = __shfl_sync(0xFFFFFFFFu, c, 0);
  uint4 qa0, qa1, qb0, qb1;
  while (c < tail_chunks) {
    std::uint32_t nc = 0;
    if (lane == 0) nc = atomicAdd(ctail, 1u);  // consumed after this chunk
    const std::uint64_t b0 = static_end + static_cast<std::uint64_t>(c) * kWChunk;
    qa0 = ld_stream(body + (b0 << 6) + lane);
    qa1 = ld_stream(body + (b0 << 6) + 32 + lane);
#pragma unroll 1
    for (std::uint64_t j = 0; j < kWChunk; j += 2) {
      qb0 = ld_stream(body + ((b0 + j + 1) << 6) + lane);
      qb1 = ld_stream(body + ((b0 + j + 1) << 6) + 32 + lane);
      code_block(qa0, qa1, b0 + j, lane, pbase, pres, sh);
      ctr.pair(qa0, qa1);
      if (j + 2 < kWChunk) {
        qa0 = ld_stream(body + ((b0 + j + 2) << 6) + lane);
        qa1 = ld_stream(body + ((b0 + j + 2) << 6) + 32 + lane);
      }
      code_block(qb0, qb1, b0 + j + 1, lane, pbase, pres, sh);
      ctr.pair(qb0, qb1);
    }
    c = __shfl_sync(0xFFFFFFFFu, nc, 0);
  }
}

template <class Ctr>
__device__ __forceinline__ void count_image_coded(const std::uint16_t* img, std::uint64_t n,
                                                  int cta, int ctas, const Ctr& ctr,
                                                  uint32_t* pbase, uint4* pres,
                                                  std::uint32_t* ctail, uint32_t sh) {
  const std::uint64_t head = head_len(img, n);
  const std::uint64_t nvec = (n - head) >> 3;
  const std::uint64_t nblk = nvec >> 6;
  const std::uint64_t tail0 = head + (nvec << 3);
  const uint4* body = reinterpret_cast<const uint4*>(img + head);
  if (cta == 0)
    for (std::uint64_t i = threadIdx.x; i < head; i += kThreads) ctr.one(img[i]);
  if (cta == ctas - 1) {
    for (std::uint64_t i = tail0 + threadIdx.x; i < n; i += kThreads) ctr.one(img[i]);
    for (std::uint64_t v = (nblk << 6) + threadIdx.x; v < nvec; v += kThreads)
      ctr.vec(ld_stream(body + v));
  }
  const uint32_t lane = threadIdx.x & 31u;
  const std::uint64_t W = static_cast<std::uint64_t>(ctas) * (kThreads / 32);
  std::uint64_t b = static_cast<std::uint64_t>(cta) * (kThreads / 32) + (threadIdx.x >> 5);
  // two register sets used in turn (no copies between stages)
  uint4 qa0, qa1, qb0, qb1;
  auto load = [&](std::uint64_t blk, uint4& x0, uint4& x1) {
    x0 = ld_stream(body + (blk << 6) + lane);
    x1 = ld_stream(body + (blk << 6) + 32 + lane);
  };
  auto work = [&](std::uint64_t blk, uint4 x0, uint4 x1) {
    code_block(x0, x1, blk, lane, pbase, pres, sh);
    ctr.pair(x0, x1);
  };
  // the last ~3% of the blocks are handed out dynamically (count_tail_coded):
  // SMs do not count at identical rates (a ~20 us first-to-last spread)
  const std::uint32_t tail_chunks = static_cast<std::uint32_t>(nblk / (32 * 8));
  const std::uint64_t static_end = nblk - static_cast<std::uint64_t>(tail_chunks) * 8;
  if (b < static_end) load(b, qa0, qa1);  // warp-uniform conditions throughout
  while (b < static_end) {
    if (b + W < static_end) load(b + W, qb0, qb1);
    work(b, qa0, qa1);
    b += W;
    if (b >= static_end) break;
    if (b + W < static_end) load(b + W, qa0, qa1);
    work(b, qb0, qb1);
    b += W;
  }
  if (tail_chunks != 0) count_tail_coded(body, static_end, tail_chunks, ctail, ctr, pbase, pres, sh);
}

// Block vectors as loaded for the apply: a narrow block's residuals (r0,
// one 16-byte load), else the two image vectors (r0, r1) -- predicated
// loads, no branch around them.
__device__ __forceinline__ void load_block(const uint4* body, const uint4* pres, std::uint64_t b,
                                           uint32_t lane, uint32_t bw, uint4& r0, uint4& r1) {
  const uint4* pr = pres + b * 32 + lane;
  const uint4* p0 = body + (b << 6) + lane;
  const uint4* p1 = p0 + 32;
  asm volatile(
      "{\n .reg .pred c;\n setp.ne.u32 c, %8, %9;\n"
      " @c ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%10];\n"
      " @!c ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%11];\n"
      " @!c ld.global.L1::no_allocate.v4.u32 {%4,%5,%6,%7}, [%12];\n}"
      : "=r"(r0.x), "=r"(r0.y), "=r"(r0.z), "=r"(r0.w), "=r"(r1.x), "=r"(r1.y), "=r"(r1.z),
        "=r"(r1.w)
      : "r"(bw), "r"(kRawBlock), "l"(pr), "l"(p0), "l"(p1));
}
__device__ __forceinline__ uint4 expand(uint32_t lo, uint32_t hi, uint32_t b2, uint32_t sh) {
  // base + (residual << sh) <= 65535 per half (sh <= 8): no carry between halves
  return make_uint4((__byte_perm(lo, 0u, 0x4140) << sh) + b2, (__byte_perm(lo, 0u, 0x4342) << sh) + b2,
                    (__byte_perm(hi, 0u, 0x4140) << sh) + b2, (__byte_perm(hi, 0u, 0x4342) << sh) + b2);
}
template <int kSwz>
__device__ __forceinline__ void store_block(const std::uint16_t* s_lut, uint4* dst, std::uint64_t b,
                                            uint32_t lane, uint32_t bw, uint4 r0, uint4 r1,
                                            uint32_t sh) {
  uint4 v0 = r0, v1 = r1;
  if (bw != kRawBlock) {
    const uint32_t b2 = bw * 0x10001u;
    v0 = expand(r0.x, r0.y, b2, sh);
    v1 = expand(r0.z, r0.w, b2, sh);
  }
  st_stream(dst + (b << 6) + lane, lookup_vec<kSwz>(s_lut, v0));
  st_stream(dst + (b << 6) + 32 + lane, lookup_vec<kSwz>(s_lut, v1));
}

// apply_image over the count pass's blocks, two per warp per stage: a
// block's base word is loaded one stage before the vectors it selects (so
// the block's loads issue as residuals or image vectors with no dependent
// wait), the next stage's loads in flight while this one is stored; the
// dynamic tail hands out chunks of 128 blocks (4 per warp).
template <int kSwz>
__device__ __forceinline__ void apply_image_coded(const std::uint16_t* s_lut,
                                                  const std::uint16_t* in, std::uint16_t* out,
                                                  std::uint64_t n, int cta, int ctas,
                                                  std::uint32_t* tail, const uint32_t* pbase,
                                                  const uint4* pres, uint32_t sh) {
  constexpr std::uint64_t kWarps = kThreads / 32;
  constexpr std::uint64_t kChunkBlk = 4 * kWarps;  // blocks per tail chunk (128 KiB of image)
  const std::uint64_t tid = static_cast<std::uint64_t>(cta) * kThreads + threadIdx.x;
  const std::uint64_t stride = static_cast<std::uint64_t>(ctas) * kThreads;
  const std::uint64_t head = head_len(in, n);
  const std::uint64_t nvec = (n - head) >> 3;
  const std::uint64_t nblk = nvec >> 6;
  const std::uint64_t tail0 = head + (nvec << 3);
  if (tid < head) out[tid] = lut_at<kSwz>(s_lut, in[tid]);
  if (tid < n - tail0) out[tail0 + tid] = lut_at<kSwz>(s_lut, in[tail0 + tid]);
  const uint4* src = reinterpret_cast<const uint4*>(in + head);
  uint4* dst = reinterpret_cast<uint4*>(out + head);
  for (std::uint64_t v = (nblk << 6) + tid; v < nvec; v += stride)
    st_stream(dst + v, lookup_vec<kSwz>(s_lut, ld_stream(src + v)));
  const uint32_t lane = threadIdx.x & 31u;
  // blocks in reverse order: the count pass coded the high blocks last, so
  // the first ones applied are partly still in L2 (~0.4% of the step)
#define MAPB(x) (nblk - 1 - (x))
  const std::uint64_t W = static_cast<std::uint64_t>(ctas) * kWarps;
  const std::uint64_t tail_chunks = 4ull * static_cast<std::uint64_t>(ctas);
  const bool dynamic = tail != nullptr && nblk >= 16 * tail_chunks * kChunkBlk;
  const std::uint64_t static_end = dynamic ? nblk - tail_chunks * kChunkBlk : nblk;
  constexpr int kU = 2;  // blocks per stage (1: 80 us slower at C3)
  std::uint64_t b = static_cast<std::uint64_t>(cta) * kWarps + (threadIdx.x >> 5);
  uint32_t bw[kU] = {}, nbw[kU] = {};
  uint4 r[kU][2], nr[kU][2];
  bool have = b + (kU - 1) * W < static_end;  // warp-uniform
  if (have) {
#pragma unroll
    for (int u = 0; u < kU; ++u) bw[u] = __ldcg(pbase + MAPB(b + u * W));
#pragma unroll
    for (int u = 0; u < kU; ++u) load_block(src, pres, MAPB(b + u * W), lane, bw[u], r[u][0], r[u][1]);
  }
  if (b + (2 * kU - 1) * W < static_end) {
#pragma unroll
    for (int u = 0; u < kU; ++u) nbw[u] = __ldcg(pbase + MAPB(b + (kU + u) * W));
  }
  while (have) {
    const std::uint64_t nx = b + kU * W;
    const bool nhave = nx + (kU - 1) * W < static_end;
    if (nhave) {
#pragma unroll
      for (int u = 0; u < kU; ++u) load_block(src, pres, MAPB(nx + u * W), lane, nbw[u], nr[u][0], nr[u][1]);
    }
    uint32_t nnbw[kU] = {};
    if (nx + (2 * kU - 1) * W < static_end) {
#pragma unroll
      for (int u = 0; u < kU; ++u) nnbw[u] = __ldcg(pbase + MAPB(nx + (kU + u) * W));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) store_block<kSwz>(s_lut, dst, MAPB(b + u * W), lane, bw[u], r[u][0], r[u][1], sh);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      r[u][0] = nr[u][0];
      r[u][1] = nr[u][1];
      bw[u] = nbw[u];
      nbw[u] = nnbw[u];
    }
    b = nx;
    have = nhave;
  }
  for (; b < static_end; b += W) {
    const uint32_t w = __ldcg(pbase + MAPB(b));
    uint4 y0, y1;
    load_block(src, pres, MAPB(b), lane, w, y0, y1);
    store_block<kSwz>(s_lut, dst, MAPB(b), lane, w, y0, y1, sh);
  }
  if (!dynamic) return;
  __shared__ std::uint32_t s_chunk;
  for (;;) {
    __syncthreads();  // the previous chunk index is consumed
    if (threadIdx.x == 0) s_chunk = atomicAdd(tail, 1u);
    __syncthreads();
    const std::uint64_t c = s_chunk;
    if (c >= tail_chunks) break;
    const std::uint64_t b0 = static_end + c * kChunkBlk + (threadIdx.x >> 5);
    uint32_t w[4];
    uint4 y[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = __ldcg(pbase + MAPB(b0 + u * kWarps));
#pragma unroll
    for (int u = 0; u < 4; ++u) load_block(src, pres, MAPB(b0 + u * kWarps), lane, w[u], y[u][0], y[u][1]);
#pragma unroll
    for (int u = 0; u < 4; ++u) store_block<kSwz>(s_lut, dst, MAPB(b0 + u * kWarps), lane, w[u], y[u][0], y[u][1], sh);
  }
}
#undef MAPB

// floor(num / d) for num < 2^53 and d >= 1 without a 64-bit integer divide
// (a ~70-instruction software sequence): num converts to f64 exactly and
// num * (1/d) carries a relative error of ~2^-52, so for the quotients here
// (<= 65535) the estimate is far within 1 of the true quotient; truncation
// is off by at most one and a single remainder test fixes it.  Bit-exact with
// the oracle's integer '/'.  Largest use: an 8-rank group of 2^32-1-sample
// bands, num < 2^35 * 65536 = 2^51.
__device__ __forceinline__ std::uint64_t udiv_exact(std::uint64_t num, std::uint64_t d,
                                                    double inv_d) {
  std::uint64_t q = static_cast<std::uint64_t>(static_cast<double>(num) * inv_d);
  const auto r = static_cast<long long>(num - q * d);
  if (r < 0) --q;
  else if (static_cast<std::uint64_t>(r) >= d) ++q;
  return q;
}

// LUT entry for bin v given the statistics (SURVEY §8a' formulas).
__device__ __forceinline__ uint32_t equalize_entry(uint32_t v,
                                                        std::uint64_t cdf,
                                                        std::uint64_t cdf_min,
                                                        std::uint64_t d, double inv_d,
                                                        uint32_t lo) {
  if (d == 0) return v;
  if (v < lo) return 0;
  return static_cast<uint32_t>(udiv_exact((cdf - cdf_min) * 65535u + d / 2, d, inv_d));
}

__device__ __forceinline__ uint32_t stretch_entry(std::uint64_t v,
                                                       std::uint64_t n,
                                                       std::uint64_t lo,
                                                       std::uint64_t hi) {
  const std::uint64_t span = hi - lo;
  if (n == 0 || span == 0) return static_cast<uint32_t>(v);
  if (v <= lo) return 0;
  if (v >= hi) return 65535;
  return static_cast<uint32_t>(
      udiv_exact((v - lo) * 65535u + span / 2, span, 1.0 / static_cast<double>(span)));
}

#ifdef GPCX_LUT_TRACE
// Phase timestamps for tools/fused_trace.cu (compiled out of the library).
__device__ unsigned long long* g_lut_trace;
#define LUT_STAMP(k)                                                          \
  do {                                                                        \
    if (threadIdx.x == 0) {                                                   \
      unsigned long long ts_;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_));                 \
      g_lut_trace[blockIdx.x * 16 + (k)] = ts_;                               \
    }                                                                         \
  } while (0)
#else
#define LUT_STAMP(k) do {} while (0)
#endif

// The equalize LUT path as ONE cooperative kernel, 1 CTA x 1024 threads per
// SM (every CTA resident); `stages` selects the phases:
//   kCount   phase 1  CTAs < nparts count their share of the image into packed
//                     smem bins and flush them as partials;        grid.sync
//            phase 2  CTA b < 128 owns bins [512b, 512b + 512): 16 groups of
//                     64 threads column-sum 1/16 of the partials each with
//                     128-bit loads (16x the memory-level parallelism of one
//                     thread per word), a smem reduction joins the groups,
//                     + overflow (zeroed for the next call) -> hist[];
//            without kCount phase 2 takes hist[] as given (multi-GPU: the
//            all-reduced histogram).  Each slice publishes (total, first,
//            last non-empty bin, count of first).
//   kBuild   grid.sync; phase 3  each slice CTA derives n, lo, hi, cdf_min and
//                     its cdf offset from the 128 summaries and writes its
//                     512 LUT entries;
//   kApply   grid.sync; phase 4  every CTA stages the LUT in smem (over the dead
//                     bins) and maps the image -- which, at C1 size, phase 1
//                     left in L2.
//   kExchange (N devices)  in phase 2, after a slice CTA has merged its 512
//            bins of this rank's band histogram (published in the rank's
//            HBM), it meets the same slice CTA of every other rank (system-
//            scope release/acquire flags, peer_rendezvous) and sums their
//            slices with P2P loads -- the histogram all-reduce, fused, one
//            slice at a time, so no grid-wide or host synchronisation.
// Single device LUT_CORRECT = kCount|kBuild|kApply, LUT_GEN = kCount|kBuild;
// N devices, one process per GPU: kCount|kExchange|kBuild|kApply (one
// launch per rank); in-process planner: kCount, then kExchange|kBuild|kApply
// after the bands' events (host-ordered, no flags); NCCL fallback:
// kCount -> all-reduce(hist) -> kBuild|kApply.  No launch gaps, and the
// partial merge is not latency-bound like a one-thread-per-bin sum.
enum Stage : int { kCount = 1, kBuild = 2, kApply = 4, kExchange = 8 };
constexpr int kSlices = kWords / 256;    // 128 CTAs own 512 bins in phases 2-3
constexpr int kGroups = kThreads / 64;   // partial groups per slice
static_assert(kGroups * 512 * 4 <= kWords * 4, "phase-2 reduction fits in the bins");
static_assert(kSlices == kFlagSlices, "one flag row per slice CTA");

__device__ __forceinline__ void st_release_sys(std::uint32_t* p, std::uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ std::uint32_t ld_acquire_sys(const std::uint32_t* p) {
  std::uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint2 ld_relaxed_sys(const uint2* p) {
  uint2 v;
  asm volatile("ld.relaxed.sys.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Device-side rendezvous of slice `slice` across the group (thread 0 of the
// slice CTA, after the CTA's words of the slice are in this rank's
// published histogram): publish seq to every rank's flag row, then wait
// for every rank's seq in our own row.  A peer that never arrives (dead
// process, mismatched seq) traps after timeout_ns instead of hanging the GPU.
__device__ void peer_rendezvous(const PeerTable* P, int slice, std::uint32_t seq,
                                unsigned long long timeout_ns) {
  const int me = P->rank, nr = P->nranks;
  __threadfence_system();
  for (int r = 0; r < nr; ++r) st_release_sys(P->flags[r] + slice * kMaxRanks + me, seq);
  const std::uint32_t* row = P->flags[me] + slice * kMaxRanks;
  const unsigned long long t0 = globaltimer_ns();
  for (int r = 0; r < nr; ++r) {
    // >= (wrap-aware): a peer may already be publishing seq + 1
    while (static_cast<int>(ld_acquire_sys(row + r) - seq) < 0) {
      __nanosleep(100);
      if (globaltimer_ns() - t0 > timeout_ns) __trap();
    }
  }
}

// Phase 2 -> phase 3 summary of one 512-bin slice.  Totals are 64-bit: one
// call's band is < 2^32 samples (its histogram is u32), but the histogram
// summed over a group of ranks can reach kMaxRanks * (2^32 - 1).
struct SliceSummary {
  unsigned long long total, first_count;  // sum of the slice's bins, count of `first`
  uint32_t first, last, pad0, pad1;       // first / last non-empty bin (0xFFFFFFFF / 0 if none)
};
static_assert(sizeof(SliceSummary) * kSlices <= kPartsOff - kBlocksOff, "summaries fit the workspace");

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
#pragma unroll
  for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, d);
  return x;
}

// Warp sum of totals: one redux.sync when they are known to fit in 32 bits
// (a single call's image, n < 2^32), the u64 shuffle tree only for a peer
// group's summed histogram (`wide`).  The redux keeps phase 3 at its
// round-1 length (~2.5 us vs ~5.8 us with the u64 tree, fused_trace).
__device__ __forceinline__ unsigned long long warp_sum_total(unsigned long long x, bool wide) {
  if (wide) return warp_sum_u64(x);
  return __reduce_add_sync(0xFFFFFFFFu, static_cast<uint32_t>(x));
}

__global__ void __launch_bounds__(kThreads, 1)
    fused_kernel(const std::uint16_t* img, std::uint16_t* out, std::uint64_t n, int nparts,
                 uint32_t* __restrict__ parts, uint32_t* __restrict__ overflow,
                 uint32_t* __restrict__ hist, SliceSummary* __restrict__ blocks, int mode,
                 std::uint16_t* __restrict__ lut, gpcx_lut_stats* __restrict__ stats,
                 int stages, const PeerTable* __restrict__ peers, std::uint32_t seq,
                 unsigned long long timeout_ns, std::uint32_t* __restrict__ tail,
                 unsigned char* __restrict__ plane) {
  extern __shared__ uint4 smem_u4[];
  uint32_t* bins = reinterpret_cast<uint32_t*>(smem_u4);
  // residual plane (kCount and kApply in this launch, room in the workspace)
  uint32_t* pbase = reinterpret_cast<uint32_t*>(plane);
  uint4* pres = reinterpret_cast<uint4*>(plane + plane_base_bytes(n));
  __shared__ unsigned long long s_wsum[8], s_wfcount[8];
  __shared__ uint32_t s_wfirst[8], s_wlast[8];
  cg::grid_group grid = cg::this_grid();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

  LUT_STAMP(0);
  const bool count = stages & kCount;
  // smem layout of this launch (the same in every CTA: a fixed sample of img)
  __shared__ uint32_t s_swz, s_wlo, s_wsh;
  if ((stages & (kCount | kApply)) != 0) sample_layout(img, n, &s_swz, &s_wlo, &s_wsh);
  if (!count) __syncthreads();  // else published by the zeroing's barrier
  // ---- phase 1: per-CTA histograms
  uint32_t* win = bins + kWords;  // the u32 window after the packed bins
  if (count && static_cast<int>(blockIdx.x) < nparts) {
    for (int i = t; i < (kWords + static_cast<int>(kWinBins)) / 4; i += kThreads)
      smem_u4[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const bool coded = plane != nullptr && (s_swz & 8u) != 0;
    const uint32_t psh = (s_swz >> 8) & 15u;  // the plane's residual shift
    auto run = [&](const auto& ctr) {
      if (coded) count_image_coded(img, n, blockIdx.x, nparts, ctr, pbase, pres, tail + 1, psh);
      else count_image(img, n, blockIdx.x, nparts, ctr);
    };
    // the window serves repetitive data too (flat / few-level images within
    // its span): red.shared of many lanes on one u32 counter runs at the
    // HBM rate (tools/hist_probe.cu mode 2), with no warp-combining probe
    const bool windowed = s_wlo != kNoWindow;
    const uint32_t lay = s_swz & 3u;
    switch (windowed ? 8u + lay : (s_swz & 7u)) {
      case 8: run(WindowCounter<0>{bins, overflow, win, s_wlo, s_wsh}); break;
      case 9: run(WindowCounter<1>{bins, overflow, win, s_wlo, s_wsh}); break;
      case 10: run(WindowCounter<2>{bins, overflow, win, s_wlo, s_wsh}); break;
      case 0: run(PlainCounter<0>{bins, overflow}); break;
      case 1: run(PlainCounter<1>{bins, overflow}); break;
      case 2: run(PlainCounter<2>{bins, overflow}); break;
      case 4: run(FewCounter<0>{bins, overflow}); break;
      case 5: run(FewCounter<1>{bins, overflow}); break;
      default: run(FewCounter<2>{bins, overflow}); break;
    }
    if (windowed) {
      __syncthreads();
      if (lay == 1) fold_window<1>(bins, overflow, win, s_wlo, s_wsh);
      else if (lay == 2) fold_window<2>(bins, overflow, win, s_wlo, s_wsh);
      else fold_window<0>(bins, overflow, win, s_wlo, s_wsh);
    }
    __syncthreads();
    LUT_STAMP(1);
    uint4* dst = reinterpret_cast<uint4*>(parts + static_cast<std::uint64_t>(blockIdx.x) * kWords);
    for (int j = t; j < kWords / 4; j += kThreads) dst[j] = smem_u4[j];
  }
  LUT_STAMP(2);
  if (count) grid.sync();
  // the coded count pass's chunk counter, zero again for the next launch
  if (count && blockIdx.x == 0 && t == 0) tail[1] = 0;
  LUT_STAMP(3);
  const uint32_t layout = s_swz & 3u;  // published by a barrier above (read only with img)

  // ---- phase 2: merge this CTA's 512-bin slice
  const bool slice_cta = static_cast<int>(blockIdx.x) < kSlices;
  const int w = blockIdx.x * 256 + t;  // word (bins 2w, 2w+1) of threads t < 256
  // bins 2w, 2w+1 of the (group's) histogram: u64 once peers are summed in
  unsigned long long c0 = 0, c1 = 0, inc = 0;
  if (slice_cta) {
    if (count) {
      const int quad = t & 63, group = t >> 6;
      const uint4* pq = reinterpret_cast<const uint4*>(parts) + blockIdx.x * 64 + quad;
      constexpr std::uint64_t kPartQuads = kWords / 4;
      uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      auto add = [&](uint4 x) {
        acc[0] += x.x & 0xFFFFu; acc[1] += x.x >> 16;
        acc[2] += x.y & 0xFFFFu; acc[3] += x.y >> 16;
        acc[4] += x.z & 0xFFFFu; acc[5] += x.z >> 16;
        acc[6] += x.w & 0xFFFFu; acc[7] += x.w >> 16;
      };
      int p = group;
      for (; p + 7 * kGroups < nparts; p += 8 * kGroups) {  // 8 loads in flight
        uint4 x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldcg(pq + (p + u * kGroups) * kPartQuads);
#pragma unroll
        for (int u = 0; u < 8; ++u) add(x[u]);
      }
      for (; p < nparts; p += kGroups) add(__ldcg(pq + p * kPartQuads));
      // red[group][bin], bin = 8 * quad + j of the slice -- logical bins:
      // in the swizzled layout the quad's physical words 4 quad .. +3 hold
      // logical words swz(.)
      if (layout != 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t pw = blockIdx.x * 256u + quad * 4u + (j >> 1);
          const uint32_t lw = layout == 1 ? swz1(pw) : swz2(pw);  // involutions
          bins[group * 512 + 2 * (lw - blockIdx.x * 256u) + (j & 1)] = acc[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) bins[group * 512 + quad * 8 + j] = acc[j];
      }
    }
    __syncthreads();
    const bool exchange = stages & kExchange;
    if (t < 256) {
      if (count) {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
          lo += bins[g * 512 + 2 * t];
          hi += bins[g * 512 + 2 * t + 1];
        }
        const uint2 ov = __ldcg(reinterpret_cast<const uint2*>(overflow) + w);
        reinterpret_cast<uint2*>(overflow)[w] = make_uint2(0, 0);
        c0 = lo + ov.x;
        c1 = hi + ov.y;
        // this band's own histogram (< 2^32 samples per call: exact in u32)
        reinterpret_cast<uint2*>(hist)[w] = make_uint2(static_cast<uint32_t>(c0),
                                                       static_cast<uint32_t>(c1));
      } else if (!exchange) {
        const uint2 h = __ldcg(reinterpret_cast<const uint2*>(hist) + w);
        c0 = h.x;
        c1 = h.y;
      }
    }
    if (exchange) {
      // multi-GPU: this slice of every rank's band histogram, summed with
      // system-scope loads of the peers' HBM (the all-reduce, fused)
      const int par = seq & 1;
      if (peers->flags[0] != nullptr) {
        __syncthreads();  // this CTA's words of the slice are published
        if (t == 0) peer_rendezvous(peers, blockIdx.x, seq, timeout_ns);
        __syncthreads();
      }
      if (t < 256) {
        const int me = count ? peers->rank : -1;  // own counts are in c0 / c1
        for (int r = 0; r < peers->nranks; ++r) {
          if (r == me) continue;
          const uint2 h = ld_relaxed_sys(reinterpret_cast<const uint2*>(peers->hist[par][r]) + w);
          c0 += h.x;
          c1 += h.y;
        }
      }
    }
    if (t < 256) {
      inc = c0 + c1;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
        if (lane >= d) inc += y;
      }
      const uint32_t first = c0 ? 2u * w : (c1 ? 2u * w + 1 : 0xFFFFFFFFu);
      const uint32_t last = c1 ? 2u * w + 1 : (c0 ? 2u * w : 0u);
      const uint32_t wfirst = __reduce_min_sync(0xFFFFFFFFu, first);
      const uint32_t wlast = __reduce_max_sync(0xFFFFFFFFu, last);
      // count of the first non-empty bin (cdf_min if it is the global one)
      const unsigned long long wfcount =
          warp_sum_u64(first == wfirst && first != 0xFFFFFFFFu ? (c0 ? c0 : c1) : 0ull);
      if (lane == 31) s_wsum[warp] = inc;
      if (lane == 0) {
        s_wfirst[warp] = wfirst;
        s_wlast[warp] = wlast;
        s_wfcount[warp] = wfcount;
      }
    }
    __syncthreads();
    if (t == 0) {
      unsigned long long sum = 0, fcount = 0;
      uint32_t first = 0xFFFFFFFFu, last = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        sum += s_wsum[i];
        if (s_wfirst[i] < first) {
          first = s_wfirst[i];
          fcount = s_wfcount[i];
        }
        last = max(last, s_wlast[i]);
      }
      // (total, first, last, count(first)): phase 3 needs no second load
      blocks[blockIdx.x] = SliceSummary{sum, fcount, first, last, 0u, 0u};
    }
  }
  LUT_STAMP(4);
  if (!(stages & kBuild)) return;
  grid.sync();
  LUT_STAMP(5);

  // ---- phase 3: LUT slice
  if (slice_cta && t < 256) {
    unsigned long long n64 = 0, off = 0, lo_count = 0;
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
    static_assert(kSlices % 32 == 0, "whole warps of slice triples");
#pragma unroll
    for (int b0 = 0; b0 < kSlices; b0 += 32) {
      const int b = b0 + lane;
      const ulonglong2 tc = __ldcg(reinterpret_cast<const ulonglong2*>(blocks + b));
      const uint2 fl = __ldcg(reinterpret_cast<const uint2*>(blocks + b) + 2);
      n64 += tc.x;
      if (b < static_cast<int>(blockIdx.x)) off += tc.x;
      if (fl.x < lo) {  // slices are disjoint: each first bin is distinct
        lo = fl.x;
        lo_count = tc.y;
      }
      if (tc.x != 0) hi = max(hi, fl.y);
    }
    const bool wide = stages & kExchange;  // peers' counts summed in: totals may exceed 2^32
    n64 = warp_sum_total(n64, wide);
    off = warp_sum_total(off, wide);
    const uint32_t my_lo = lo;
    lo = __reduce_min_sync(0xFFFFFFFFu, lo);
    hi = __reduce_max_sync(0xFFFFFFFFu, hi);
    const unsigned long long cdf_min64 = warp_sum_total(my_lo == lo ? lo_count : 0ull, wide);
    unsigned long long warp_off = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < warp) warp_off += s_wsum[i];
    const uint32_t v0 = 2u * w;
    uint32_t e0, e1;
    if (lo == 0xFFFFFFFFu) {  // empty image: identity LUT, zero stats
      e0 = v0;
      e1 = v0 + 1;
      if (w == 0) *stats = gpcx_lut_stats{0, 0, 0, 0};
    } else {
      const std::uint64_t nn = n64;
      const std::uint64_t cdf_min = cdf_min64;
      if (w == 0) *stats = gpcx_lut_stats{nn, lo, hi, mode == GPCX_LUT_STRETCH ? 0 : cdf_min};
      if (mode == GPCX_LUT_STRETCH) {
        e0 = stretch_entry(v0, nn, lo, hi);
        e1 = stretch_entry(v0 + 1, nn, lo, hi);
      } else {
        const std::uint64_t d = nn - cdf_min;
        const double inv_d = d != 0 ? 1.0 / static_cast<double>(d) : 0.0;
        const std::uint64_t cdf1 = static_cast<std::uint64_t>(off) + warp_off + inc;
        e0 = equalize_entry(v0, cdf1 - c1, cdf_min, d, inv_d, lo);
        e1 = equalize_entry(v0 + 1, cdf1, cdf_min, d, inv_d, lo);
      }
    }
    reinterpret_cast<uint32_t*>(lut)[w] = e0 | (e1 << 16);
  }
  LUT_STAMP(6);
  if (!(stages & kApply)) return;
  if (blockIdx.x == 0 && t == 0) *tail = 0;  // apply's dynamic tail, published by the sync
  grid.sync();
  LUT_STAMP(7);

  // ---- phase 4: apply
  const auto* s_lut = reinterpret_cast<const std::uint16_t*>(smem_u4);
  if (layout == 1) stage_lut<1>(smem_u4, lut);
  else if (layout == 2) stage_lut<2>(smem_u4, lut);
  else stage_lut<0>(smem_u4, lut);
  __syncthreads();
  LUT_STAMP(8);
  const uint32_t psh = (s_swz >> 8) & 15u;
  if (plane != nullptr && (s_swz & 8u) != 0) {  // the plane this launch's count pass coded
    if (layout == 1) apply_image_coded<1>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail, pbase, pres, psh);
    else if (layout == 2) apply_image_coded<2>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail, pbase, pres, psh);
    else apply_image_coded<0>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail, pbase, pres, psh);
  } else {
    if (layout == 1) apply_image<1>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail);
    else if (layout == 2) apply_image<2>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail);
    else apply_image<0>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail);
  }
#ifdef GPCX_LUT_TRACE
  __syncthreads();
#endif
  LUT_STAMP(9);
}

__device__ __forceinline__ void minmax_vec(uint4 q, uint32_t& mn2,
                                           uint32_t& mx2) {
  mn2 = __vminu2(mn2, __vminu2(__vminu2(q.x, q.y), __vminu2(q.z, q.w)));
  mx2 = __vmaxu2(mx2, __vmaxu2(__vmaxu2(q.x, q.y), __vmaxu2(q.z, q.w)));
}

// Per-CTA (lo, hi) of the samples; SIMD u16x2 min/max per thread, then
// redux.sync warp reductions and a 32-entry smem step.
__global__ void __launch_bounds__(kThreads)
    minmax_kernel(const std::uint16_t* __restrict__ img, std::uint64_t n,
                  uint2* __restrict__ slots) {
  __shared__ uint32_t smn[32], smx[32];
  uint32_t mn2 = 0xFFFFFFFFu, mx2 = 0;
  const std::uint64_t head = head_len(img, n);
  const std::uint64_t nvec = (n - head) >> 3;
  const std::uint64_t tail0 = head + (nvec << 3);
  const std::uint64_t tid = static_cast<std::uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * kThreads;
  if (tid < head) {
    const uint32_t v = img[tid];
    mn2 = __vminu2(mn2, v | (v << 16));
    mx2 = __vmaxu2(mx2, v | (v << 16));
  }
  if (tid < n - tail0) {
    const uint32_t v = img[tail0 + tid];
    mn2 = __vminu2(mn2, v | (v << 16));
    mx2 = __vmaxu2(mx2, v | (v << 16));
  }
  const uint4* body = reinterpret_cast<const uint4*>(img + head);
  std::uint64_t i = tid;
  for (; i + (kUnroll - 1) * stride < nvec; i += kUnroll * stride) {
    uint4 q[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) q[u] = ld_stream(body + i + u * stride);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) minmax_vec(q[u], mn2, mx2);
  }
  for (; i < nvec; i += stride) minmax_vec(ld_stream(body + i), mn2, mx2);

  uint32_t mn = min(mn2 & 0xFFFFu, mn2 >> 16);
  uint32_t mx = max(mx2 & 0xFFFFu, mx2 >> 16);
  mn = __reduce_min_sync(0xFFFFFFFFu, mn);
  mx = __reduce_max_sync(0xFFFFFFFFu, mx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    smn[warp] = mn;
    smx[warp] = mx;
  }
  __syncthreads();
  if (warp == 0) {
    mn = __reduce_min_sync(0xFFFFFFFFu, smn[lane]);
    mx = __reduce_max_sync(0xFFFFFFFFu, smx[lane]);
    if (lane == 0) slots[blockIdx.x] = make_uint2(mn, mx);
  }
}

__global__ void __launch_bounds__(1024)
    minmax_reduce_kernel(const uint2* __restrict__ slots, int nslots,
                         std::uint64_t n, gpcx_lut_stats* __restrict__ stats) {
  __shared__ uint32_t smn[32], smx[32];
  uint32_t mn = 0xFFFFFFFFu, mx = 0;
  for (int i = threadIdx.x; i < nslots; i += 1024) {
    const uint2 s = slots[i];
    mn = min(mn, s.x);
    mx = max(mx, s.y);
  }
  mn = __reduce_min_sync(0xFFFFFFFFu, mn);
  mx = __reduce_max_sync(0xFFFFFFFFu, mx);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    smn[warp] = mn;
    smx[warp] = mx;
  }
  __syncthreads();
  if (warp == 0) {
    mn = __reduce_min_sync(0xFFFFFFFFu, smn[lane]);
    mx = __reduce_max_sync(0xFFFFFFFFu, smx[lane]);
    if (lane == 0) {
      if (n == 0) *stats = gpcx_lut_stats{0, 0, 0, 0};
      else *stats = gpcx_lut_stats{n, mn, mx, 0};
    }
  }
}

// Stretch LUT from (lo, hi): 32 CTAs x 1024 threads, two entries (one u32
// store) per thread -- one CTA doing all 65536 took 11 us of the stretch step.
__global__ void __launch_bounds__(1024)
    from_minmax_kernel(const gpcx_lut_stats* __restrict__ stats,
                       std::uint16_t* __restrict__ lut) {
  const std::uint64_t n = stats->n;
  const std::uint64_t lo = stats->lo, hi = stats->hi;
  const uint32_t w = blockIdx.x * 1024 + threadIdx.x;  // entries 2w, 2w + 1
  reinterpret_cast<uint32_t*>(lut)[w] =
      stretch_entry(2 * w, n, lo, hi) | (stretch_entry(2 * w + 1, n, lo, hi) << 16);
}

// out = LUT[in].  The 128 KiB LUT is staged once per CTA in shared memory
// (1 CTA/SM, persistent grid); the image streams through with 128-bit
// loads/stores, kUnroll vectors in flight per thread.
__global__ void __launch_bounds__(kThreads, 1)
    apply_kernel(const std::uint16_t* __restrict__ lut_g,
                 const std::uint16_t* in, std::uint16_t* out, std::uint64_t n,
                 int vector_ok) {
  extern __shared__ uint4 smem_u4[];
  __shared__ uint32_t s_swz;
  sample_layout(in, n, &s_swz);
  __syncthreads();
  const uint32_t layout = s_swz & 3u;
  if (layout == 1) stage_lut<1>(smem_u4, lut_g);
  else if (layout == 2) stage_lut<2>(smem_u4, lut_g);
  else stage_lut<0>(smem_u4, lut_g);
  __syncthreads();
  const std::uint16_t* s_lut = reinterpret_cast<const std::uint16_t*>(smem_u4);
  if (!vector_ok) {  // mismatched alignment of in/out: scalar path
    const std::uint64_t tid = static_cast<std::uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
    for (std::uint64_t i = tid; i < n; i += static_cast<std::uint64_t>(gridDim.x) * kThreads)
      out[i] = layout == 1 ? lut_at<1>(s_lut, in[i])
                           : (layout == 2 ? lut_at<2>(s_lut, in[i]) : lut_at<0>(s_lut, in[i]));
    return;
  }
  if (layout == 1) apply_image<1>(s_lut, in, out, n, blockIdx.x, gridDim.x);
  else if (layout == 2) apply_image<2>(s_lut, in, out, n, blockIdx.x, gridDim.x);
  else apply_image<0>(s_lut, in, out, n, blockIdx.x, gridDim.x);
}

// LUT_CORRECT stretch in ONE cooperative launch (1 CTA x 1024 threads per
// SM) instead of min/max + reduce + LUT + apply: per-CTA min/max of the
// image -> grid sync -> every CTA reduces the slots and builds the whole
// stretch LUT straight into its own smem (64 entries per thread, no second
// grid-wide step; CTA b also stores 1024-word slices b, b + grid, ... of
// the caller's LUT, CTA 0 the stats) -> apply.  Same entries as
// from_minmax_kernel (stretch_entry), so bit-identical.
template <int kSwz>
__device__ __forceinline__ void build_stretch_lut(uint32_t* s_words, std::uint16_t* lut_g,
                                                  std::uint64_t n, std::uint64_t lo,
                                                  std::uint64_t hi) {
#pragma unroll 4
  for (int k = 0; k < kWords / kThreads; ++k) {
    const uint32_t w = static_cast<uint32_t>(k * kThreads) + threadIdx.x;
    const uint32_t e = stretch_entry(2 * w, n, lo, hi) | (stretch_entry(2 * w + 1, n, lo, hi) << 16);
    s_words[phys_word<kSwz>(w)] = e;
    if (k % static_cast<int>(gridDim.x) == static_cast<int>(blockIdx.x))
      reinterpret_cast<uint32_t*>(lut_g)[w] = e;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    stretch_fused_kernel(const std::uint16_t* img, std::uint16_t* out,  // may alias (in place)
                         std::uint64_t n, uint2* __restrict__ slots, std::uint16_t* lut_g,
                         gpcx_lut_stats* stats, std::uint32_t* __restrict__ tail) {
  extern __shared__ uint4 smem_u4[];
  __shared__ uint32_t smn[32], smx[32], s_swz;
  cg::grid_group grid = cg::this_grid();
  sample_layout(img, n, &s_swz);
  uint32_t mn2 = 0xFFFFFFFFu, mx2 = 0;
  {
    const std::uint64_t head = head_len(img, n);
    const std::uint64_t nvec = (n - head) >> 3;
    const std::uint64_t tail0 = head + (nvec << 3);
    const std::uint64_t tid = static_cast<std::uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * kThreads;
    if (tid < head) {
      const uint32_t v = img[tid];
      mn2 = __vminu2(mn2, v | (v << 16));
      mx2 = __vmaxu2(mx2, v | (v << 16));
    }
    if (tid < n - tail0) {
      const uint32_t v = img[tail0 + tid];
      mn2 = __vminu2(mn2, v | (v << 16));
      mx2 = __vmaxu2(mx2, v | (v << 16));
    }
    const uint4* body = reinterpret_cast<const uint4*>(img + head);
    std::uint64_t i = tid;
    for (; i + (kUnroll - 1) * stride < nvec; i += kUnroll * stride) {
      uint4 q[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) q[u] = ld_stream(body + i + u * stride);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) minmax_vec(q[u], mn2, mx2);
    }
    for (; i < nvec; i += stride) minmax_vec(ld_stream(body + i), mn2, mx2);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t mn = __reduce_min_sync(0xFFFFFFFFu, min(mn2 & 0xFFFFu, mn2 >> 16));
  uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, max(mx2 & 0xFFFFu, mx2 >> 16));
  if (lane == 0) {
    smn[warp] = mn;
    smx[warp] = mx;
  }
  __syncthreads();
  if (warp == 0) {
    mn = __reduce_min_sync(0xFFFFFFFFu, smn[lane]);
    mx = __reduce_max_sync(0xFFFFFFFFu, smx[lane]);
    if (lane == 0) slots[blockIdx.x] = make_uint2(mn, mx);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *tail = 0;  // apply's dynamic tail
  grid.sync();
  if (warp == 0) {
    mn = 0xFFFFFFFFu;
    mx = 0;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) {
      const uint2 sl = __ldcg(slots + b);
      mn = min(mn, sl.x);
      mx = max(mx, sl.y);
    }
    mn = __reduce_min_sync(0xFFFFFFFFu, mn);
    mx = __reduce_max_sync(0xFFFFFFFFu, mx);
    if (lane == 0) {
      smn[0] = mn;
      smx[0] = mx;
      if (blockIdx.x == 0) *stats = gpcx_lut_stats{n, mn, mx, 0};
    }
  }
  __syncthreads();
  const std::uint64_t lo = smn[0], hi = smx[0];
  const uint32_t layout = s_swz & 3u;
  uint32_t* s_words = reinterpret_cast<uint32_t*>(smem_u4);
  if (layout == 1) build_stretch_lut<1>(s_words, lut_g, n, lo, hi);
  else if (layout == 2) build_stretch_lut<2>(s_words, lut_g, n, lo, hi);
  else build_stretch_lut<0>(s_words, lut_g, n, lo, hi);
  __syncthreads();
  const std::uint16_t* s_lut = reinterpret_cast<const std::uint16_t*>(smem_u4);
  if (layout == 1) apply_image<1>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail);
  else if (layout == 2) apply_image<2>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail);
  else apply_image<0>(s_lut, img, out, n, blockIdx.x, gridDim.x, tail);
}

bool g_attrs_set[64] = {};

void set_attrs_once() {
  int dev = 0;
  GPCX_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && g_attrs_set[dev]) return;
  GPCX_CUDA(cudaFuncSetAttribute(fused_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemHist));
  GPCX_CUDA(cudaFuncSetAttribute(apply_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLut));
  GPCX_CUDA(cudaFuncSetAttribute(stretch_fused_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLut));
  if (dev < 64) g_attrs_set[dev] = true;
}

}  // namespace

uint32_t* ws_hist(void* ws) {
  return reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(ws) + kHistOff);
}

std::uint64_t workspace_bytes() {
  return kPartsOff + static_cast<std::uint64_t>(kMaxParts) * kWords * 4;
}

std::uint64_t plane_bytes(std::uint64_t n) {
  return n >= kPlaneMin ? plane_base_bytes(n) + (n >> 9) * 512 : 0;
}

std::uint64_t workspace_bytes(std::uint64_t n) { return workspace_bytes() + plane_bytes(n); }

int parts_for(std::uint64_t n, int num_sms) {
  // One CTA per SM once there is enough work; at least 64 Ki samples per
  // CTA below that so the per-CTA partial flush stays amortised.
  const std::uint64_t want = (n + 65535) / 65536;
  int p = static_cast<int>(std::min<std::uint64_t>(want, static_cast<std::uint64_t>(num_sms)));
  return std::max(1, std::min(p, kMaxParts));
}

namespace {
// fused_kernel over the whole device (see its comment for `stages`).
// GPCX_LUT_PLANE=0: never code the residual plane (A/B only).
bool plane_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("GPCX_LUT_PLANE");
    return v == nullptr || v[0] != '0';
  }();
  return on;
}

void launch_fused(int stages, const std::uint16_t* img, std::uint16_t* out, std::uint64_t n,
                  uint32_t* hist, int mode, std::uint16_t* lut, gpcx_lut_stats* stats, void* ws,
                  cudaStream_t stream, const PeerTable* peers = nullptr, std::uint32_t seq = 0,
                  unsigned long long timeout_ns = 0, std::uint64_t ws_bytes = 0) {
  set_attrs_once();
  auto* base = static_cast<unsigned char*>(ws);
  // the residual plane, given a plane-sized workspace: count and apply in
  // this launch, or a split pair (launch_hist -> launch_correct_from_peers
  // on one workspace and image, the in-process planner) -- an apply-only
  // launch handed ws_bytes reads the plane its count launch wrote
  unsigned char* plane = nullptr;
  if ((stages & (kCount | kApply)) != 0 && plane_bytes(n) != 0 &&
      ws_bytes >= workspace_bytes(n) && plane_enabled())
    plane = base + workspace_bytes();
  auto* overflow = reinterpret_cast<uint32_t*>(base + kOverflowOff);
  auto* parts = reinterpret_cast<uint32_t*>(base + kPartsOff);
  auto* blocks = reinterpret_cast<SliceSummary*>(base + kBlocksOff);
  auto* tail = reinterpret_cast<std::uint32_t*>(base + kTailOff);
  if (hist == nullptr) hist = reinterpret_cast<uint32_t*>(base + kHistOff);
  const int sms = device_sm_count();
  int nparts = parts_for(n, sms);
  void* args[] = {const_cast<std::uint16_t**>(&img), &out, &n, &nparts, &parts, &overflow,
                  &hist, &blocks, &mode, &lut, &stats, &stages,
                  const_cast<PeerTable**>(&peers), &seq, &timeout_ns, &tail, &plane};
  GPCX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fused_kernel),
                                        dim3(std::max(sms, kSlices)), dim3(kThreads), args,
                                        kSmemHist, stream));
}

// GPCX_LUT_STRETCH_FUSED=0: the four-launch stretch path (A/B only).
bool stretch_fused_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("GPCX_LUT_STRETCH_FUSED");
    return v == nullptr || v[0] != '0';
  }();
  return on;
}

bool co_aligned(const void* a, const void* b) {
  return ((reinterpret_cast<std::uintptr_t>(a) ^ reinterpret_cast<std::uintptr_t>(b)) & 15u) == 0;
}
}  // namespace

void launch_hist(const std::uint16_t* img, std::uint64_t n, uint32_t* hist,
                 void* ws, cudaStream_t stream, std::uint64_t ws_bytes) {
  launch_fused(kCount, img, nullptr, n, hist, GPCX_LUT_EQUALIZE, nullptr, nullptr, ws, stream,
               nullptr, 0, 0, ws_bytes);
}

void launch_from_hist(const uint32_t* hist, int mode, std::uint16_t* lut,
                      gpcx_lut_stats* stats, void* ws, cudaStream_t stream) {
  launch_fused(kBuild, nullptr, nullptr, 0, const_cast<uint32_t*>(hist), mode, lut, stats, ws,
               stream);
}

void launch_correct_from_hist(const uint32_t* hist, int mode, const std::uint16_t* in,
                              std::uint16_t* out, std::uint64_t n, std::uint16_t* lut,
                              gpcx_lut_stats* stats, void* ws, cudaStream_t stream) {
  if (co_aligned(in, out) && n != 0) {
    launch_fused(kBuild | kApply, in, out, n, const_cast<uint32_t*>(hist), mode, lut, stats, ws,
                 stream);
    return;
  }
  launch_from_hist(hist, mode, lut, stats, ws, stream);
  launch_apply(lut, in, out, n, stream);
}

void launch_hist_lut(const std::uint16_t* img, std::uint64_t n, int mode, std::uint16_t* lut,
                     gpcx_lut_stats* stats, void* ws, cudaStream_t stream) {
  launch_fused(kCount | kBuild, img, nullptr, n, nullptr, mode, lut, stats, ws, stream);
}

void launch_correct(const std::uint16_t* in, std::uint16_t* out, std::uint64_t n, int mode,
                    std::uint16_t* lut, gpcx_lut_stats* stats, void* ws, cudaStream_t stream,
                    std::uint64_t ws_bytes) {
  if (mode == GPCX_LUT_EQUALIZE && co_aligned(in, out) && n != 0) {
    launch_fused(kCount | kBuild | kApply, in, out, n, nullptr, mode, lut, stats, ws, stream,
                 nullptr, 0, 0, ws_bytes);
    return;
  }
  if (mode == GPCX_LUT_STRETCH && co_aligned(in, out) && n != 0 && stretch_fused_enabled()) {
    set_attrs_once();
    auto* slots = reinterpret_cast<uint2*>(static_cast<unsigned char*>(ws) + kMinMaxOff);
    auto* tail = reinterpret_cast<std::uint32_t*>(static_cast<unsigned char*>(ws) + kTailOff);
    const int sms = device_sm_count();
    void* args[] = {const_cast<std::uint16_t**>(&in), &out, &n, &slots, &lut, &stats, &tail};
    GPCX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(stretch_fused_kernel),
                                          dim3(sms), dim3(kThreads), args, kSmemLut, stream));
    return;
  }
  if (mode == GPCX_LUT_EQUALIZE) {
    launch_hist_lut(in, n, mode, lut, stats, ws, stream);
  } else {
    launch_minmax(in, n, stats, ws, stream);
    launch_from_minmax(stats, lut, stream);
  }
  launch_apply(lut, in, out, n, stream);
}

void launch_correct_peer(const PeerTable* table, std::uint32_t* own_hist, std::uint32_t seq,
                         std::uint64_t timeout_ns, const std::uint16_t* in, std::uint16_t* out,
                         std::uint64_t n, int mode, std::uint16_t* lut, gpcx_lut_stats* stats,
                         void* ws, cudaStream_t stream, std::uint64_t ws_bytes) {
  // every rank launches the same stages (the rendezvous sits in phase 2);
  // the apply needs co-aligned in/out (the callers check) or out == nullptr
  const bool fused_apply = out != nullptr && co_aligned(in, out);
  const int stages = kCount | kExchange | kBuild | (fused_apply ? kApply : 0);
  launch_fused(stages, in, fused_apply ? out : nullptr, n, own_hist, mode, lut, stats, ws,
               stream, table, seq, timeout_ns, fused_apply ? ws_bytes : 0);
  if (out != nullptr && !fused_apply) launch_apply(lut, in, out, n, stream);
}

void launch_correct_from_peers(const PeerTable* table, std::uint32_t seq, int mode,
                               const std::uint16_t* in, std::uint16_t* out, std::uint64_t n,
                               std::uint16_t* lut, gpcx_lut_stats* stats, void* ws,
                               cudaStream_t stream, std::uint64_t ws_bytes) {
  if (out == nullptr || n == 0) {
    launch_fused(kExchange | kBuild, nullptr, nullptr, 0, nullptr, mode, lut, stats, ws, stream,
                 table, seq, 0);
    return;
  }
  if (co_aligned(in, out)) {
    launch_fused(kExchange | kBuild | kApply, in, out, n, nullptr, mode, lut, stats, ws, stream,
                 table, seq, 0, ws_bytes);
    return;
  }
  launch_fused(kExchange | kBuild, nullptr, nullptr, 0, nullptr, mode, lut, stats, ws, stream,
               table, seq, 0);
  launch_apply(lut, in, out, n, stream);
}

void launch_minmax(const std::uint16_t* img, std::uint64_t n,
                   gpcx_lut_stats* stats, void* ws, cudaStream_t stream) {
  auto* slots = reinterpret_cast<uint2*>(static_cast<unsigned char*>(ws) + kMinMaxOff);
  const int p = std::min(kMaxParts, std::max(1, static_cast<int>(std::min<std::uint64_t>(
                                                    (n + 65535) / 65536,
                                                    static_cast<std::uint64_t>(2 * device_sm_count())))));
  minmax_kernel<<<p, kThreads, 0, stream>>>(img, n, slots);
  GPCX_LAUNCH_CHECK();
  minmax_reduce_kernel<<<1, 1024, 0, stream>>>(slots, p, n, stats);
  GPCX_LAUNCH_CHECK();
}

void launch_from_minmax(const gpcx_lut_stats* stats, std::uint16_t* lut,
                        cudaStream_t stream) {
  from_minmax_kernel<<<kWords / 1024, 1024, 0, stream>>>(stats, lut);
  GPCX_LAUNCH_CHECK();
}

void launch_apply(const std::uint16_t* lut, const std::uint16_t* in,
                  std::uint16_t* out, std::uint64_t n, cudaStream_t stream) {
  if (n == 0) return;
  set_attrs_once();
  const int vector_ok =
      ((reinterpret_cast<std::uintptr_t>(in) ^ reinterpret_cast<std::uintptr_t>(out)) & 15u) == 0;
  const std::uint64_t want = (n + 8191) / 8192;
  const int p = static_cast<int>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>(want, static_cast<std::uint64_t>(device_sm_count()))));
  apply_kernel<<<p, kThreads, kSmemLut, stream>>>(lut, in, out, n, vector_ok);
  GPCX_LAUNCH_CHECK();
}

}  // namespace lut
}  // namespace gpcx
