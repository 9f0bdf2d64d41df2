// gpc_b200_tasks.cpp -- see gpc_b200_tasks.hpp.
#include "gpc_b200_tasks.hpp"

#include <algorithm>
#include <string>
#include <vector>

#include "gpc/tasks.hpp"
#include "gpcx.h"

namespace gpc::task {

namespace {

// gpcx_status = 1 + Errc ordinal (include/gpcx.h), so the reference's own
// response_code() mapping applies unchanged.
void check(int rc) {
  if (rc != GPCX_OK) throw Error(static_cast<Errc>(rc - 1), gpcx_last_error());
}

TaskDescriptor b200_descriptor(const std::string& flag) {
  TaskDescriptor d;
  d.flag = flag;
  char req[256] = {};
  check(gpcx_required_params(flag.c_str(), req, sizeof(req)));
  for (std::string list = req; !list.empty();) {
    const std::size_t comma = list.find(',');
    d.required_params.push_back(list.substr(0, comma));
    list = comma == std::string::npos ? "" : list.substr(comma + 1);
  }
  d.payload_rule = [flag](const wire::ParamMap& params) {
    std::uint64_t len = 0;
    check(gpcx_payload_len(flag.c_str(), params.serialize().c_str(), &len));
    return len;
  };
  d.handler = [flag](const wire::ParamMap& params, std::span<const std::uint8_t> payload) {
    const std::string text = params.serialize();
    std::uint64_t want = 0;
    check(gpcx_output_len(flag.c_str(), text.c_str(), &want));
    TaskOutput out;
    out.payload.resize(want);
    std::uint64_t got = 0;
    char result[wire::kParamsSize + 1] = {};
    check(gpcx_run(flag.c_str(), text.c_str(), payload.data(), payload.size(), out.payload.data(),
                   out.payload.size(), &got, result, sizeof(result)));
    out.payload.resize(got);
    out.params = wire::ParamMap::parse(result);
    return out;
  };
  return d;
}

}  // namespace

void add_b200_tasks(TaskRegistry& registry) {
  char flags[512] = {};
  check(gpcx_flags(flags, sizeof(flags)));
  const std::vector<std::string> have = registry.flags();
  for (std::string list = flags; !list.empty();) {
    const std::size_t comma = list.find(',');
    const std::string flag = list.substr(0, comma);
    if (std::find(have.begin(), have.end(), flag) == have.end())
      registry.add(b200_descriptor(flag));
    list = comma == std::string::npos ? "" : list.substr(comma + 1);
  }
}

TaskRegistry make_b200_registry(const par::ExecPlan& plan) {
  TaskRegistry out;
  add_b200_tasks(out);
  const TaskRegistry cpu = make_builtin_registry(plan);
  const std::vector<std::string> gpu = out.flags();
  for (const std::string& flag : cpu.flags())
    if (std::find(gpu.begin(), gpu.end(), flag) == gpu.end()) out.add(cpu.lookup(flag));
  return out;
}

}  // namespace gpc::task
