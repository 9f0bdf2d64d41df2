// task_spec.cpp -- see task_spec.hpp.
#include "task_spec.hpp"

namespace gpcx::task {

Flag flag_of(std::string_view flag) {
  if (flag == "LUT_GEN") return Flag::LutGen;
  if (flag == "LUT_APPLY") return Flag::LutApply;
  if (flag == "LUT_CORRECT") return Flag::LutCorrect;
  if (flag == "MATMUL") return Flag::Matmul;
  if (flag == "BAYER_BILINEAR") return Flag::BayerBilinear;
  if (flag == "BAYER_GRADIENT") return Flag::BayerGradient;
  if (flag == "DEVINFO") return Flag::DevInfo;
  if (flag == "LSQ_POLYFIT") return Flag::LsqPolyfit;
  fail(Errc::UnknownTask, std::string(flag));
}

const char* flag_name(Flag f) {
  switch (f) {
    case Flag::LutGen: return "LUT_GEN";
    case Flag::LutApply: return "LUT_APPLY";
    case Flag::LutCorrect: return "LUT_CORRECT";
    case Flag::Matmul: return "MATMUL";
    case Flag::BayerBilinear: return "BAYER_BILINEAR";
    case Flag::BayerGradient: return "BAYER_GRADIENT";
    case Flag::DevInfo: return "DEVINFO";
    case Flag::LsqPolyfit: return "LSQ_POLYFIT";
  }
  return "?";
}

// Sorted like the registry's std::map iteration order.
std::vector<Flag> all_flags() {
  return {Flag::BayerBilinear, Flag::BayerGradient, Flag::DevInfo,    Flag::LsqPolyfit,
          Flag::LutApply,      Flag::LutCorrect,    Flag::LutGen,     Flag::Matmul};
}

std::vector<std::string> required_params(Flag f) {
  if (f == Flag::Matmul) return {"m", "k", "n"};
  if (f == Flag::DevInfo) return {};
  if (f == Flag::LsqPolyfit) return {"lines", "pixels", "order"};
  return {"rows", "cols"};
}

LsqParams parse_lsq(const wire::ParamMap& params) {
  LsqParams p;
  p.lines = params.get_uint("lines");
  p.pixels = params.get_uint("pixels");
  const std::uint64_t order = params.get_uint("order");
  if (order > 8)
    fail(Errc::OrderTooHigh, "order " + std::to_string(order) + " exceeds 8");
  p.order = static_cast<int>(order);
  const std::string dtype = params.get_or("dtype", "f64");
  if (dtype == "f32") p.f32 = true;
  else if (dtype != "f64") fail(Errc::BadValue, "dtype=" + dtype);
  return p;
}

const char* mode_name(int mode) { return mode == GPCX_LUT_STRETCH ? "stretch" : "equalize"; }

const char* prec_name(int prec) {
  switch (prec) {
    case GPCX_PREC_TF32: return "tf32";
    case GPCX_PREC_BF16: return "bf16";
    default: return "f32";
  }
}

const char* phase_name(int phase) {
  static const char* const kNames[4] = {"RGGB", "BGGR", "GRBG", "GBRG"};
  return kNames[phase & 3];
}

namespace {
// Dimension check of a synthetic request: nothing crosses the wire, so the
// bound is the kernels' (fewer than 2^32 elements), not the 1 GiB cap.
std::uint64_t synth_elems(std::string_view a_key, std::uint64_t a, std::string_view b_key,
                          std::uint64_t b) {
  if (a == 0 || b == 0)
    fail(Errc::BadValue, std::string(a == 0 ? a_key : b_key) + " must be positive");
  if (a >= (1ull << 32) || b >= (1ull << 32) || a * b >= (1ull << 32))
    fail(Errc::Overflow, std::string(a_key) + "*" + std::string(b_key) +
                             " must stay below 2^32 elements");
  return a * b;
}
}  // namespace

SynthParams parse_synth(Flag f, const wire::ParamMap& params) {
  SynthParams s;
  if (!params.has("synth")) return s;
  const std::string kind = params.get("synth");
  s.on = true;
  if (f == Flag::LutGen || f == Flag::LutCorrect) {
    if (kind == "ramp12") s.kind = GPCX_IMG_RAMP12;
    else if (kind == "uniform16") s.kind = GPCX_IMG_UNIFORM16;
    else fail(Errc::BadValue, "synth=" + kind);
  } else if (f == Flag::Matmul) {
    if (kind == "exact8") s.kind = GPCX_MAT_EXACT8;
    else if (kind == "uniform32") s.kind = GPCX_MAT_UNIFORM32;
    else fail(Errc::BadValue, "synth=" + kind);
    if (params.has("samples")) s.samples = params.get_uint("samples");
    if (s.samples == 0 || s.samples > (1ull << 20))
      fail(Errc::BadValue, "samples must be 1 .. 1048576");
  } else {
    fail(Errc::BadValue, std::string("synth= is not supported by ") + flag_name(f));
  }
  if (params.has("seed")) s.seed = params.get_uint("seed");
  return s;
}

LutParams parse_lut(Flag f, const wire::ParamMap& params) {
  LutParams p;
  p.rows = params.get_uint("rows");
  p.cols = params.get_uint("cols");
  if (params.has("synth") && f == Flag::LutApply)
    fail(Errc::BadValue, "synth= is not supported by LUT_APPLY (its LUT is an input)");
  if (params.has("synth"))
    synth_elems("rows", p.rows, "cols", p.cols);
  else
    wire::dim_product("rows", p.rows, "cols", p.cols, 2);  // validates + caps
  const std::string dtype = params.get_or("dtype", "u16");
  if (dtype != "u16") fail(Errc::BadValue, "dtype=" + dtype);
  if (f != Flag::LutApply) {
    const std::string mode = params.get_or("mode", "equalize");
    if (mode == "equalize") p.mode = GPCX_LUT_EQUALIZE;
    else if (mode == "stretch") p.mode = GPCX_LUT_STRETCH;
    else fail(Errc::BadValue, "mode=" + mode);
  }
  return p;
}

MatmulParams parse_matmul(const wire::ParamMap& params) {
  MatmulParams p;
  p.m = params.get_uint("m");
  p.k = params.get_uint("k");
  p.n = params.get_uint("n");
  if (params.has("synth")) {
    synth_elems("m", p.m, "k", p.k);
    synth_elems("k", p.k, "n", p.n);
    synth_elems("m", p.m, "n", p.n);
  } else {
    const std::uint64_t a_bytes = wire::dim_product("m", p.m, "k", p.k, 4);
    const std::uint64_t b_bytes = wire::dim_product("k", p.k, "n", p.n, 4);
    wire::capped_sum(a_bytes, b_bytes);
    wire::dim_product("m", p.m, "n", p.n, 4);  // the response must fit too
  }
  const std::string prec = params.get_or("prec", "f32");
  if (prec == "f32") p.prec = GPCX_PREC_F32;
  else if (prec == "tf32") p.prec = GPCX_PREC_TF32;
  else if (prec == "bf16") p.prec = GPCX_PREC_BF16;
  else fail(Errc::BadValue, "prec=" + prec);
  return p;
}

// Same order of checks as the reference handler run_demosaic
// (proj/src/tasks.cpp:16-21): rows, cols, dtype, then phase.
BayerParams parse_bayer(const wire::ParamMap& params) {
  BayerParams p;
  p.rows = params.get_uint("rows");
  p.cols = params.get_uint("cols");
  wire::dim_product("rows", p.rows, "cols", p.cols, 2);
  const std::string dtype = params.get_or("dtype", "u16");
  if (dtype != "u16") fail(Errc::BadValue, "dtype=" + dtype);
  const std::string phase = params.get_or("phase", "RGGB");
  if (phase == "RGGB") p.phase = 0;
  else if (phase == "BGGR") p.phase = 1;
  else if (phase == "GRBG") p.phase = 2;
  else if (phase == "GBRG") p.phase = 3;
  else fail(Errc::BadValue, "phase=" + phase);
  return p;
}

std::uint64_t payload_len(Flag f, const wire::ParamMap& params) {
  switch (f) {
    case Flag::LutGen:
    case Flag::LutCorrect: {
      const LutParams p = parse_lut(f, params);
      return parse_synth(f, params).on ? 0 : p.pixels() * 2;
    }
    case Flag::LutApply: {
      const LutParams p = parse_lut(f, params);
      return wire::capped_sum(kLutBytes, p.pixels() * 2);
    }
    case Flag::Matmul: {
      const MatmulParams p = parse_matmul(params);
      return parse_synth(f, params).on ? 0 : (p.m * p.k + p.k * p.n) * 4;
    }
    case Flag::BayerBilinear:
    case Flag::BayerGradient: {
      // sized like expected_payload_len's BAYER_* rule (wire.cpp:207-211):
      // dims only; dtype / phase are the handler's to reject.
      const std::uint64_t rows = params.get_uint("rows");
      const std::uint64_t cols = params.get_uint("cols");
      return wire::dim_product("rows", rows, "cols", cols, 2);
    }
    case Flag::DevInfo:
      return 0;
    case Flag::LsqPolyfit: {
      // expected_payload_len's LSQ_POLYFIT rule (wire.cpp:212-224): dtype is
      // checked here, before the payload, order only by the handler.
      const std::uint64_t lines = params.get_uint("lines");
      const std::uint64_t pixels = params.get_uint("pixels");
      const std::string dtype = params.get_or("dtype", "f64");
      std::uint64_t scale = 0;
      if (dtype == "f32") scale = 4;
      else if (dtype == "f64") scale = 8;
      else fail(Errc::BadValue, "dtype=" + dtype);
      return wire::dim_product("lines", lines, "pixels", pixels, scale);
    }
  }
  return 0;
}

std::uint64_t output_len(Flag f, const wire::ParamMap& params) {
  switch (f) {
    case Flag::LutGen:
      parse_lut(f, params);
      return kLutBytes;
    case Flag::LutApply:
      return parse_lut(f, params).pixels() * 2;
    case Flag::LutCorrect: {
      const LutParams p = parse_lut(f, params);
      return parse_synth(f, params).on ? 8 : p.pixels() * 2;
    }
    case Flag::Matmul: {
      const MatmulParams p = parse_matmul(params);
      const SynthParams s = parse_synth(f, params);
      return s.on ? s.samples * kSynthSampleBytes : p.m * p.n * 4;
    }
    case Flag::BayerBilinear:
    case Flag::BayerGradient: {
      const BayerParams p = parse_bayer(params);
      return p.rows * p.cols * 6;
    }
    case Flag::DevInfo:
      return 0;
    case Flag::LsqPolyfit: {
      const LsqParams p = parse_lsq(params);
      return p.lines * (static_cast<std::uint64_t>(p.order) + 2) * 8;
    }
  }
  return 0;
}

}  // namespace gpcx::task
