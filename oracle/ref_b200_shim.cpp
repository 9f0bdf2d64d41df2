// ref_b200_shim.cpp -- TEST INFRASTRUCTURE.  The REFERENCE server with the
// B200 plugin (integration/gpc_b200_tasks.cpp) registered next to its
// built-in tasks -- the drop-in INTEGRATION.md describes -- built from the
// reference's own sources into oracle/_ref/libgpc_b200_ref.so and linked
// to libgpcx.so.  tests/test_integration.py drives it.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "gpc/devinfo.hpp"
#include "gpc/error.hpp"
#include "gpc/server.hpp"
#include "gpc/tasks.hpp"
#include "gpc_b200_tasks.hpp"

using namespace gpc;

namespace {

thread_local std::string g_err;

const task::TaskRegistry& registry() {
  static const task::TaskRegistry* r = [] {
    auto devices = std::make_shared<task::DeviceList>();
    devinfo::DeviceInfo d;
    d.name = "Test Device";
    devices->push_back(d);
    auto* reg = new task::TaskRegistry(task::make_builtin_registry(par::ExecPlan{}, devices));
    task::add_b200_tasks(*reg);
    return reg;
  }();
  return *r;
}

struct Handle {
  std::unique_ptr<srv::Server> server;
};

}  // namespace

extern "C" {

const char* refb_last_error(void) { return g_err.c_str(); }

int refb_flags(char* out, std::size_t cap) {
  try {
    std::string s;
    for (const auto& f : registry().flags()) s += (s.empty() ? "" : ",") + f;
    std::strncpy(out, s.c_str(), cap - 1);
    out[cap - 1] = 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int refb_handle_request(const std::uint8_t* req, std::size_t len, std::uint8_t* resp,
                        std::size_t cap, std::size_t* resp_len) {
  try {
    wire::MemoryStream stream(std::vector<std::uint8_t>(req, req + len));
    srv::handle_connection(stream, registry());
    const auto& w = stream.written();
    *resp_len = w.size();
    if (w.size() > cap) return 24;
    std::memcpy(resp, w.data(), w.size());
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  }
}

int refb_server_start(int max_tasks, void** handle, std::uint16_t* port) {
  try {
    auto h = std::make_unique<Handle>();
    srv::ServerConfig cfg;
    cfg.bind_addr = "127.0.0.1";
    cfg.port = 0;
    cfg.max_tasks = max_tasks;
    h->server = std::make_unique<srv::Server>(cfg, registry());
    h->server->start();
    *port = h->server->port();
    *handle = h.release();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  }
}

int refb_server_stop(void* handle) {
  auto* h = static_cast<Handle*>(handle);
  h->server->stop();
  delete h;
  return 0;
}

}  // extern "C"

// A second reference registry built with make_b200_registry: every flag
// libgpcx serves (BAYER_*, DEVINFO included) on the GPU, LSQ_POLYFIT on the CPU.
namespace {
const gpc::task::TaskRegistry& registry_gpu_first() {
  static const gpc::task::TaskRegistry* r =
      new gpc::task::TaskRegistry(gpc::task::make_b200_registry(gpc::par::ExecPlan{}));
  return *r;
}
}  // namespace

extern "C" int refb2_flags(char* out, std::size_t cap) {
  std::string s;
  for (const auto& f : registry_gpu_first().flags()) s += (s.empty() ? "" : ",") + f;
  std::strncpy(out, s.c_str(), cap - 1);
  out[cap - 1] = 0;
  return 0;
}

extern "C" int refb2_handle_request(const std::uint8_t* req, std::size_t len, std::uint8_t* resp,
                                    std::size_t cap, std::size_t* resp_len) {
  try {
    gpc::wire::MemoryStream stream(std::vector<std::uint8_t>(req, req + len));
    gpc::srv::handle_connection(stream, registry_gpu_first());
    const auto& w = stream.written();
    *resp_len = w.size();
    if (w.size() > cap) return 24;
    std::memcpy(resp, w.data(), w.size());
    return 0;
  } catch (const gpc::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  }
}
