// registry.hpp -- the task plugin contract of the B200 executor.
//
// Same shape as the reference's gpc::task (proj/include/gpc/registry.hpp:23-78):
// a TaskDescriptor {flag, required_params, payload_rule, handler}, a
// TaskRegistry with add/lookup/flags, a never-throwing dispatch() that maps
// every failure onto the closed ERR:<CODE> set, sanitize_message() and
// make_response_frame().  One extension for zero-copy staging: a handler's
// TaskOutput may carry its payload in a pinned pooled buffer (`pinned`)
// instead of a std::vector, so the response goes from the D2H target
// straight to the socket without the reference's copy at registry.cpp:129.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "runtime.hpp"
#include "wire.hpp"

namespace gpcx::task {

struct TaskOutput {
  wire::ParamMap params;              // bytes= is added by dispatch
  std::vector<std::uint8_t> payload;  // reference-style payload, or
  rt::PinnedLease pinned;             // zero-copy payload of pinned_len bytes
  std::uint64_t pinned_len = 0;
  std::span<const std::uint8_t> bytes() const {
    if (pinned.get() != nullptr)
      return {static_cast<const std::uint8_t*>(pinned.get()), pinned_len};
    return payload;
  }
};

using PayloadRule = std::function<std::uint64_t(const wire::ParamMap&)>;
using Handler =
    std::function<TaskOutput(const wire::ParamMap&, std::span<const std::uint8_t>)>;

struct TaskDescriptor {
  std::string flag;
  std::vector<std::string> required_params;
  PayloadRule payload_rule;
  Handler handler;
};

class TaskRegistry {
 public:
  void add(TaskDescriptor descriptor);  // FieldTooLong / InvalidCharacter / BadValue / DuplicateFlag
  const TaskDescriptor& lookup(std::string_view flag) const;  // UnknownTask
  std::vector<std::string> flags() const;

 private:
  std::map<std::string, TaskDescriptor, std::less<>> tasks_;
};

std::string response_code(Errc code);

struct DispatchResult {
  std::string status;  // "OK" or "ERR:<CODE>"
  wire::ParamMap params;
  TaskOutput output;   // payload (empty on error)
  bool ok() const { return status == "OK"; }
  std::span<const std::uint8_t> payload() const { return output.bytes(); }
};

// Request whose payload may live outside a Frame (e.g. a pinned buffer).
struct RequestView {
  const wire::TaskHeader* header;
  std::span<const std::uint8_t> payload;
};

// The one parse of a request header: descriptor lookup,
// params, required keys, payload length from the descriptor's rule and the
// marker check -- what the reference does twice, in handle_connection
// (proj/src/server.cpp:73-93) and again in dispatch (registry.cpp:83-90).
// The front end admits a request once, sizes its staging from
// payload_len, and runs it with run_admitted.  Throws gpcx::Error.
struct Admission {
  const TaskDescriptor* descriptor = nullptr;
  wire::ParamMap params;
  std::uint64_t payload_len = 0;
};
Admission admit(const TaskRegistry& registry, const wire::TaskHeader& header);

// Runs an admitted request's handler on its payload; never throws (every
// failure becomes ERR:<CODE>, proj/src/registry.cpp:98-120).
DispatchResult run_admitted(const Admission& admission, std::span<const std::uint8_t> payload);

// A failure result: ERR:<CODE> with the sanitised msg= (no payload).
DispatchResult error_result(Errc code, std::string_view what);

// admit + run_admitted (the reference's dispatch contract, one parse).
DispatchResult dispatch(const TaskRegistry& registry, const RequestView& request);
inline DispatchResult dispatch(const TaskRegistry& registry, const wire::Frame& request) {
  return dispatch(registry, RequestView{&request.header, request.payload});
}

std::string sanitize_message(std::string_view text, const wire::ParamMap& existing);

// Response header for a result: status in the flag slot, marker from the
// payload, output_name echoed when it encodes.
wire::TaskHeader make_response_header(const DispatchResult& result, std::string_view output_name);

// The GPU tasks of task_spec.hpp as descriptors whose handlers run on the
// bound B200s (exec::execute) and answer from pinned buffers.
TaskRegistry make_b200_registry();

}  // namespace gpcx::task
