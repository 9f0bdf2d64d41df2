// executor.hpp -- runs one GPU task request: the body behind gpcx_run and
// the server's handlers.  The reference equivalent is a TaskDescriptor
// handler: params -> decode -> kernel -> encode -> result params
// (proj/src/tasks.cpp:13-35); here it is params -> H2D (async, per-request
// stream) -> sm_100a kernels -> D2H, with the multi-GPU shard/gather planner
// deciding how many devices take part.
#pragma once

#include <cstdint>
#include <span>
#include <string>

#include "task_spec.hpp"
#include "wire.hpp"

namespace gpcx::exec {

// `in` / `out` are host memory (pinned or pageable).  out.size() must be at
// least task::output_len().  Returns the result params (without bytes=).
wire::ParamMap execute(task::Flag flag, const wire::ParamMap& params,
                       std::span<const std::uint8_t> in, std::span<std::uint8_t> out);
// The same for a request the registry already admitted (task::admit): its
// payload length was checked there, so it is not recomputed.
wire::ParamMap execute_admitted(task::Flag flag, const wire::ParamMap& params,
                                std::span<const std::uint8_t> in, std::span<std::uint8_t> out);

// The same, on typed host buffers and without the wire's 1 GiB cap (the
// in-process entry points gpcx_lut_host / gpcx_matmul_host).
// With `synth` on, the image is generated on the devices (img == nullptr)
// and LUT_CORRECT returns the corrected image's position-keyed digest in
// *digest instead of the pixels (out == nullptr).
gpcx_lut_stats lut_host(task::Flag flag, const task::LutParams& p, const std::uint16_t* img,
                        const std::uint16_t* lut_in, std::uint16_t* out,
                        std::uint16_t* lut_out, const task::SynthParams* synth = nullptr,
                        std::uint64_t* digest = nullptr);
void matmul_host(const task::MatmulParams& p, const float* A, const float* B, float* C);
// A synthetic MATMUL: A / B generated on the devices, `samples` entries of
// C written to `out` as (u32 row, u32 col, f32 value) LE (task_spec.hpp).
void matmul_synth(const task::MatmulParams& p, const task::SynthParams& synth, std::uint8_t* out);
// BAYER_BILINEAR / BAYER_GRADIENT on host buffers (out: 3 planes).
void bayer_host(bool gradient, const task::BayerParams& p, const std::uint16_t* in,
                std::uint16_t* out);
// LSQ_POLYFIT on host buffers: out = lines x (order + 2) doubles.
void lsq_host(const task::LsqParams& p, const void* y, double* out);
// DEVINFO document of the bound devices (probed once) and its device count.
const std::string& devinfo_xml();
std::uint64_t devinfo_count();

// Work size (pixels or output rows) below which a request stays on one
// device even when several are bound.
inline constexpr std::uint64_t kShardMinPixels = 1ull << 24;
inline constexpr std::uint64_t kShardMinFlops = 1ull << 36;

}  // namespace gpcx::exec
