// cuda_util.hpp -- CUDA error plumbing: every CUDA failure becomes
// gpcx::Error(TaskFailed), i.e. ERR:TASK_FAILED on the wire (SURVEY §5:
// "map cudaError_t to Errc::TaskFailed").  There is no CPU fallback.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "status.hpp"

namespace gpcx::rt {
// Device health bookkeeping (host/runtime.cpp): quarantines the current
// device when `e` is a sticky error.
void note_cuda_error(cudaError_t e, const char* where);
}  // namespace gpcx::rt

#define GPCX_STR2_(x) #x
#define GPCX_STR_(x) GPCX_STR2_(x)
#define GPCX_CUDA(call)                                                  \
  do {                                                                   \
    const cudaError_t gpcx_err_ = (call);                                \
    if (gpcx_err_ != cudaSuccess) {                                      \
      ::gpcx::rt::note_cuda_error(gpcx_err_, __FILE__ ":" GPCX_STR_(__LINE__)); \
      ::gpcx::fail(::gpcx::Errc::TaskFailed,                             \
                   std::string("CUDA: ") + cudaGetErrorString(gpcx_err_) + \
                       " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
    }                                                                    \
  } while (0)

// Launch-error check right after a <<<>>> launch.
#define GPCX_LAUNCH_CHECK() GPCX_CUDA(cudaGetLastError())
