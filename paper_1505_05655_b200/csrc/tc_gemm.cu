// tc_gemm.cu -- tensor-core (tcgen05) MATMUL path, prec = tf32 | bf16.
// Placeholder until the TMA + tcgen05 kernel lands: fails loudly (no
// fallback to another path).
#include <cstdint>

#include "cuda_util.hpp"
#include "kernels.hpp"

namespace gpcx::gemm {

std::uint64_t tc_workspace_bytes(int, std::uint64_t, std::uint64_t, std::uint64_t) { return 0; }

void launch_tc(int, std::uint64_t, std::uint64_t, std::uint64_t, const float*, std::uint64_t,
               const float*, std::uint64_t, float*, std::uint64_t, void*, cudaStream_t) {
  fail(Errc::TaskFailed, "tensor-core MATMUL path not built yet");
}

}  // namespace gpcx::gemm
