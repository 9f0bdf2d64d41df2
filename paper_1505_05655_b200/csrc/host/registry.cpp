// registry.cpp -- see registry.hpp.  The error mapping and message rules are
// pinned against the reference's dispatch (proj/src/registry.cpp:38-140) by
// tests/test_executor.py.
#include "registry.hpp"

#include <algorithm>

#include "executor.hpp"
#include "task_spec.hpp"

namespace gpcx::task {

namespace {
bool printable(char c) {
  const auto b = static_cast<unsigned char>(c);
  return b >= 0x20 && b <= 0x7E;
}
}  // namespace

void TaskRegistry::add(TaskDescriptor d) {
  if (d.flag.empty() || d.flag.size() > wire::kTaskFlagSize)
    fail(Errc::FieldTooLong, "task flag '" + d.flag + "'");
  if (!std::all_of(d.flag.begin(), d.flag.end(), printable))
    fail(Errc::InvalidCharacter, "task flag '" + d.flag + "'");
  if (!d.payload_rule || !d.handler)
    fail(Errc::BadValue, "descriptor for '" + d.flag + "' lacks a payload rule or handler");
  if (tasks_.find(d.flag) != tasks_.end()) fail(Errc::DuplicateFlag, d.flag);
  std::string key = d.flag;
  tasks_.emplace(std::move(key), std::move(d));
}

const TaskDescriptor& TaskRegistry::lookup(std::string_view flag) const {
  const auto it = tasks_.find(flag);
  if (it == tasks_.end()) fail(Errc::UnknownTask, std::string(flag));
  return it->second;
}

std::vector<std::string> TaskRegistry::flags() const {
  std::vector<std::string> out;
  for (const auto& kv : tasks_) out.push_back(kv.first);
  return out;
}

std::string response_code(Errc code) { return gpcx::response_code(code); }

std::string sanitize_message(std::string_view text, const wire::ParamMap& existing) {
  const std::size_t used = existing.serialize().size();
  const std::size_t overhead = (used == 0 ? 0 : 1) + 4;  // "," + "msg="
  const std::size_t budget =
      wire::kParamsSize > used + overhead ? wire::kParamsSize - used - overhead : 0;
  std::string msg;
  msg.reserve(std::min(budget, text.size()));
  for (char c : text) {
    if (msg.size() >= budget) break;
    msg += printable(c) ? c : '?';
  }
  return msg;
}

Admission admit(const TaskRegistry& registry, const wire::TaskHeader& h) {
  Admission a;
  a.descriptor = &registry.lookup(h.task_flag);
  a.params = wire::ParamMap::parse(h.params);
  for (const std::string& key : a.descriptor->required_params)
    if (!a.params.has(key)) fail(Errc::MissingParam, key);
  a.payload_len = a.descriptor->payload_rule(a.params);
  const bool marked = h.data_marker == wire::kMarkerData;
  if (marked && a.payload_len == 0)
    fail(Errc::PayloadMismatch, "marker promises payload, expected length 0");
  if (!marked && a.payload_len > 0)
    fail(Errc::PayloadMismatch,
         "no payload marker, expected " + std::to_string(a.payload_len) + " bytes");
  return a;
}

namespace {
DispatchResult failure(const std::string& code, const char* what) {
  DispatchResult r;
  r.status = "ERR:" + code;
  r.params.set("msg", sanitize_message(what, r.params));
  return r;
}
}  // namespace

DispatchResult error_result(Errc code, std::string_view what) {
  return failure(gpcx::response_code(code), std::string(what).c_str());
}

DispatchResult run_admitted(const Admission& a, std::span<const std::uint8_t> payload) {
  try {
    if (payload.size() != a.payload_len)
      fail(Errc::PayloadMismatch, "payload is " + std::to_string(payload.size()) +
                                      " bytes, want " + std::to_string(a.payload_len));
    DispatchResult r;
    r.output = a.descriptor->handler(a.params, payload);
    r.params = std::move(r.output.params);
    r.output.params = wire::ParamMap();
    r.params.set("bytes", static_cast<std::uint64_t>(r.output.bytes().size()));
    r.status = "OK";
    return r;
  } catch (const Error& e) {
    return failure(gpcx::response_code(e.code()), e.what());
  } catch (const std::exception& e) {
    return failure("TASK_FAILED", e.what());
  } catch (...) {
    return failure("TASK_FAILED", "unknown failure");
  }
}

DispatchResult dispatch(const TaskRegistry& registry, const RequestView& request) {
  Admission a;
  try {
    a = admit(registry, *request.header);
  } catch (const Error& e) {
    return failure(gpcx::response_code(e.code()), e.what());
  } catch (const std::exception& e) {
    return failure("TASK_FAILED", e.what());
  }
  return run_admitted(a, request.payload);
}

wire::TaskHeader make_response_header(const DispatchResult& result, std::string_view output_name) {
  wire::TaskHeader h;
  h.task_flag = result.status;
  h.data_marker = result.payload().empty() ? wire::kMarkerNone : wire::kMarkerData;
  h.params = result.params.serialize();
  const bool echo = output_name.size() <= wire::kOutputNameSize &&
                    std::all_of(output_name.begin(), output_name.end(), printable);
  if (echo) h.output_name = std::string(output_name);
  return h;
}

TaskRegistry make_b200_registry() {
  TaskRegistry registry;
  for (const Flag f : all_flags()) {
    TaskDescriptor d;
    d.flag = flag_name(f);
    d.required_params = required_params(f);
    d.payload_rule = [f](const wire::ParamMap& p) { return payload_len(f, p); };
    d.handler = [f](const wire::ParamMap& p, std::span<const std::uint8_t> in) {
      TaskOutput out;
      const std::uint64_t len =
          f == Flag::DevInfo ? exec::devinfo_xml().size() : output_len(f, p);
      out.pinned = rt::pinned_acquire(len);
      out.pinned_len = len;
      // admitted: payload length already checked against this rule
      out.params = exec::execute_admitted(
          f, p, in, std::span<std::uint8_t>(static_cast<std::uint8_t*>(out.pinned.get()), len));
      return out;
    };
    registry.add(std::move(d));
  }
  return registry;
}

}  // namespace gpcx::task
