// task_spec.hpp -- the GPU task flags: required params, payload / output
// sizing and parameter parsing.  These are the TaskDescriptor pieces the
// reference's built-in tasks define in proj/src/tasks.cpp:64-123 (sized_by ->
// expected_payload_len, proj/src/wire.cpp:205-227), for the flags of
// SURVEY.md §8a' plus the §8f "next" rows:
//
//   flag            required     payload in                 payload out
//   LUT_GEN         rows, cols   rows*cols u16 LE           65536 u16 LE (LUT)
//   LUT_APPLY       rows, cols   LUT (131072 B) || image    rows*cols u16 LE
//   LUT_CORRECT     rows, cols   rows*cols u16 LE           rows*cols u16 LE
//   MATMUL          m, k, n      A (m*k f32) || B (k*n f32) C (m*n f32)
//   BAYER_BILINEAR  rows, cols   rows*cols u16 LE mosaic    R || G || B planes
//   BAYER_GRADIENT  rows, cols   rows*cols u16 LE mosaic    R || G || B planes
//   DEVINFO         -            -                          XML text
//
// Optional: dtype=u16 and mode=equalize|stretch (LUT_GEN / LUT_CORRECT);
// prec=f32|tf32|bf16 (MATMUL); dtype=u16, phase=RGGB|BGGR|GRBG|GBRG
// (BAYER_*, as proj/src/tasks.cpp:13-35).  Sizes follow the reference's
// dim_product() rules and the 1 GiB kMaxPayload cap.
//
// Header-only synthetic requests (SURVEY.md §8d option ii): with
// synth=ramp12|uniform16 (LUT_GEN, LUT_CORRECT) or synth=exact8|uniform32
// (MATMUL) and optional seed=S (default 24301 = 0x5eed) the request carries
// NO payload (marker 0x00): the inputs are generated on the GPUs by the
// counter-based generators (the same bits the oracle generates), so the
// over-cap configs C3 / C4 run through the served path.  The 1 GiB cap then
// bounds only the response:
//   LUT_GEN     -> the LUT (131072 B), rows*cols < 2^32
//   LUT_CORRECT -> 8 bytes: the position-keyed u64 digest of the corrected
//                  image, sum_i splitmix64((i << 16) | out[i]) mod 2^64
//   MATMUL      -> samples=N (default 4096, <= 2^20) entries of C, each
//                  (u32 row, u32 col, f32 value) LE; entry j is at
//                  row = splitmix64(seed ^ 2j) mod m, col = splitmix64(seed ^
//                  (2j+1)) mod n; A uses seed, B splitmix64(seed); m*k, k*n and
//                  m*n < 2^32 elements each.
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "../../../include/gpcx.h"
#include "wire.hpp"

namespace gpcx::task {

//   LSQ_POLYFIT     lines, pixels, lines*pixels f32/f64 LE  per line a_0..a_m, SSE (f64)
//                   order
enum class Flag {
  LutGen, LutApply, LutCorrect, Matmul, BayerBilinear, BayerGradient, DevInfo, LsqPolyfit
};

inline constexpr std::uint64_t kLutBytes = 65536 * 2;

Flag flag_of(std::string_view flag);  // UnknownTask
const char* flag_name(Flag f);
std::vector<Flag> all_flags();
std::vector<std::string> required_params(Flag f);

struct LutParams {
  std::uint64_t rows = 0, cols = 0;
  int mode = GPCX_LUT_EQUALIZE;
  std::uint64_t pixels() const { return rows * cols; }
};
struct MatmulParams {
  std::uint64_t m = 0, k = 0, n = 0;
  int prec = GPCX_PREC_F32;
};
struct BayerParams {
  std::uint64_t rows = 0, cols = 0;
  int phase = 0;  // gpc::img::CfaPhase ordinal: RGGB, BGGR, GRBG, GBRG
};

struct SynthParams {
  bool on = false;
  int kind = 0;  // GPCX_IMG_* (LUT) or GPCX_MAT_* (MATMUL)
  std::uint64_t seed = 0x5EED;
  std::uint64_t samples = 4096;  // MATMUL only
};
inline constexpr std::uint64_t kSynthSampleBytes = 12;  // u32 row, u32 col, f32 value

struct LsqParams {
  std::uint64_t lines = 0, pixels = 0;
  int order = 0;
  bool f32 = false;
};

// Parse + validate (MissingParam / BadValue / Overflow).
LutParams parse_lut(Flag f, const wire::ParamMap& params);
// The reference handler's order (proj/src/tasks.cpp:37-60): lines, pixels,
// order (OrderTooHigh above 8), dtype.
LsqParams parse_lsq(const wire::ParamMap& params);
MatmulParams parse_matmul(const wire::ParamMap& params);
// synth= / seed= / samples= (BadValue for a flag or kind that has none).
SynthParams parse_synth(Flag f, const wire::ParamMap& params);
BayerParams parse_bayer(const wire::ParamMap& params);

std::uint64_t payload_len(Flag f, const wire::ParamMap& params);
// DEVINFO's output length depends on the device list: callers use
// exec::devinfo_xml() directly.
std::uint64_t output_len(Flag f, const wire::ParamMap& params);

const char* mode_name(int mode);
const char* prec_name(int prec);
const char* phase_name(int phase);

}  // namespace gpcx::task
