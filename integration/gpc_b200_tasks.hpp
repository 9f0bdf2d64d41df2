// gpc_b200_tasks.hpp -- reference-side plugin for the B200 backend.
//
// Drop this file and gpc_b200_tasks.cpp into the reference tree
// (proj/src/) and link libgpcx.so: the reference server then serves
// LUT_GEN / LUT_APPLY / LUT_CORRECT / MATMUL on the GPUs through the C ABI
// of include/gpcx.h, registered exactly like the built-in tasks
// (proj/src/tasks.cpp:64-123).  See INTEGRATION.md.
#pragma once

#include "gpc/registry.hpp"

namespace gpc::task {

// Adds the four GPU task descriptors (payload_rule -> gpcx_payload_len,
// handler -> gpcx_output_len + gpcx_run).  Throws DuplicateFlag if a flag
// is already registered; every gpcx failure is rethrown as the gpc::Error
// with the same Errc, so dispatch() maps it to the same ERR:<CODE>.
void add_b200_tasks(TaskRegistry& registry);

}  // namespace gpc::task
