// gpc_b200_tasks.hpp -- reference-side plugin for the B200 backend.
//
// Drop this file and gpc_b200_tasks.cpp into the reference tree
// (proj/src/) and link libgpcx.so: the reference server then serves
// LUT_GEN / LUT_APPLY / LUT_CORRECT / MATMUL on the GPUs through the C ABI
// of include/gpcx.h, registered exactly like the built-in tasks
// (proj/src/tasks.cpp:64-123).  See INTEGRATION.md.
#pragma once

#include "gpc/parexec.hpp"
#include "gpc/registry.hpp"

namespace gpc::task {

// Adds the GPU task descriptors (payload_rule -> gpcx_payload_len, handler
// -> gpcx_output_len + gpcx_run) for every flag libgpcx serves that the
// registry does not hold yet -- called at the end of make_builtin_registry
// it adds LUT_GEN / LUT_APPLY / LUT_CORRECT / MATMUL and leaves the
// built-in CPU BAYER_* / DEVINFO in place.  Every gpcx failure is rethrown
// as the gpc::Error with the same Errc, so dispatch() maps it to the same
// ERR:<CODE>.
void add_b200_tasks(TaskRegistry& registry);

// A registry where every flag libgpcx serves runs on the GPUs (including
// BAYER_BILINEAR / BAYER_GRADIENT / DEVINFO) and the remaining built-ins
// (LSQ_POLYFIT) stay on the CPU -- use it in place of make_builtin_registry.
TaskRegistry make_b200_registry(const par::ExecPlan& plan);

}  // namespace gpc::task
