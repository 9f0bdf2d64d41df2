// trace.hpp -- NVTX ranges for the request phases (SURVEY.md §5 tracing:
// the reference only has the per-connection log line, proj/src/
// server.cpp:37-47).  Ranges live in the "gpcx" NVTX domain:
//   request  (async: accept -> connection closed, spans threads)
//   receive | h2d | kernel | d2h | task | send  (per thread, nested)
// so an Nsight Systems / ncu --nvtx capture shows where each request's time
// goes on the host and on the stream.  NVTX3 is header-only; with no tool
// attached every call is a branch on a null function pointer.
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace gpcx::obs {

inline nvtxDomainHandle_t domain() {
  static const nvtxDomainHandle_t d = nvtxDomainCreateA("gpcx");
  return d;
}

inline nvtxEventAttributes_t attrs(const char* name) {
  nvtxEventAttributes_t a{};
  a.version = NVTX_VERSION;
  a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
  a.messageType = NVTX_MESSAGE_TYPE_ASCII;
  a.message.ascii = name;
  return a;
}

// Thread-scoped range (push / pop on the calling thread).
class Range {
 public:
  explicit Range(const char* name) {
    const nvtxEventAttributes_t a = attrs(name);
    nvtxDomainRangePushEx(domain(), &a);
  }
  ~Range() { nvtxDomainRangePop(domain()); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};

// Range that may end on another thread (a request's life in the server).
class AsyncRange {
 public:
  AsyncRange() = default;
  ~AsyncRange() { end(); }
  AsyncRange(const AsyncRange&) = delete;
  AsyncRange& operator=(const AsyncRange&) = delete;
  void start(const char* name) {
    end();
    const nvtxEventAttributes_t a = attrs(name);
    id_ = nvtxDomainRangeStartEx(domain(), &a);
    open_ = true;
  }
  void end() {
    if (open_) nvtxDomainRangeEnd(domain(), id_);
    open_ = false;
  }

 private:
  nvtxRangeId_t id_ = 0;
  bool open_ = false;
};

}  // namespace gpcx::obs
