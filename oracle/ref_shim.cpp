// ref_shim.cpp -- TEST INFRASTRUCTURE.  A C-ABI window onto the reference
// implementation, compiled together with the reference's OWN sources
// (/root/reference/proj/src/*.cpp, proj/reference/*.cpp -- compiled where
// they lie, never copied) into oracle/_ref/libgpc_ref.so by oracle/Makefile.
//
// It lets the Python tests run the real reference on the same inputs as the
// B200 backend: wire codec, ParamMap, dispatch / handle_connection, the TCP
// server and client, the demosaic kernels and their independent gpcref
// oracles.  It also registers the CPU restatement of the LUT / MATMUL tasks
// (oracle/gpcx_oracle.c) into a reference TaskRegistry -- the "reference
// CPU path" of SURVEY.md §8d: the restated kernels served through the
// reference's own dispatch and server code.  bench.py --impl reference and
// the cpu_baseline leg time that path.
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "gpc/client.hpp"
#include "gpc/demosaic.hpp"
#include "gpc/devinfo.hpp"
#include "gpc/error.hpp"
#include "gpc/lsq.hpp"
#include "gpc/registry.hpp"
#include "gpc/server.hpp"
#include "gpc/tasks.hpp"
#include "gpc/wire.hpp"
#include "gpcx.h"
#include "gpcx_oracle.h"
#include "reference.hpp"

using namespace gpc;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return static_cast<int>(Errc::TaskFailed) + 1;
  }
}

void put(const std::string& s, char* out, std::size_t cap) {
  if (out == nullptr || cap == 0) return;
  const std::size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
  std::memcpy(out, s.data(), n);
  out[n] = 0;
}

// ---- oracle task descriptors (CPU restatement behind reference dispatch) ----

constexpr std::uint64_t kLutBytes = 131072;

struct LutArgs {
  std::uint64_t rows, cols;
  int mode;
};

// The sizing rules and messages of the product's task_spec.cpp, written
// against the reference's own ParamMap: the reference's dim_product()
// (proj/src/wire.cpp:67-80) is file-local, so it is restated here.
std::uint64_t dims(const char* ak, std::uint64_t a, const char* bk, std::uint64_t b,
                   std::uint64_t scale) {
  if (a == 0) fail(Errc::BadValue, std::string(ak) + " must be positive");
  if (b == 0) fail(Errc::BadValue, std::string(bk) + " must be positive");
  if (a > wire::kMaxPayload || b > wire::kMaxPayload)
    fail(Errc::Overflow, "dimension exceeds payload cap");
  const std::uint64_t len = a * b * scale;
  if (len > wire::kMaxPayload)
    fail(Errc::Overflow, "payload length " + std::to_string(len) + " exceeds cap " +
                             std::to_string(wire::kMaxPayload));
  return len;
}

std::uint64_t capped(std::uint64_t a, std::uint64_t b) {
  const std::uint64_t len = a + b;
  if (len > wire::kMaxPayload)
    fail(Errc::Overflow, "payload length " + std::to_string(len) + " exceeds cap " +
                             std::to_string(wire::kMaxPayload));
  return len;
}

LutArgs lut_args(const wire::ParamMap& p, bool has_mode) {
  LutArgs a{p.get_uint("rows"), 0, ORC_LUT_EQUALIZE};
  a.cols = p.get_uint("cols");
  dims("rows", a.rows, "cols", a.cols, 2);
  const std::string dtype = p.get_or("dtype", "u16");
  if (dtype != "u16") fail(Errc::BadValue, "dtype=" + dtype);
  if (has_mode) {
    const std::string mode = p.get_or("mode", "equalize");
    if (mode == "stretch") a.mode = ORC_LUT_STRETCH;
    else if (mode != "equalize") fail(Errc::BadValue, "mode=" + mode);
  }
  return a;
}

struct MatArgs {
  std::uint64_t m, k, n;
  int prec;
};

MatArgs mat_args(const wire::ParamMap& p) {
  MatArgs a{p.get_uint("m"), 0, 0, ORC_PREC_F32};
  a.k = p.get_uint("k");
  a.n = p.get_uint("n");
  const std::uint64_t la = dims("m", a.m, "k", a.k, 4);
  const std::uint64_t lb = dims("k", a.k, "n", a.n, 4);
  capped(la, lb);
  dims("m", a.m, "n", a.n, 4);
  const std::string prec = p.get_or("prec", "f32");
  if (prec == "tf32") a.prec = ORC_PREC_TF32;
  else if (prec == "bf16") a.prec = ORC_PREC_BF16;
  else if (prec != "f32") fail(Errc::BadValue, "prec=" + prec);
  return a;
}

void lut_result(task::TaskOutput& out, const LutArgs& a, const orc_lut_stats& st) {
  out.params.set("rows", a.rows);
  out.params.set("cols", a.cols);
  out.params.set("mode", a.mode == ORC_LUT_STRETCH ? "stretch" : "equalize");
  out.params.set("lo", static_cast<std::uint64_t>(st.lo));
  out.params.set("hi", static_cast<std::uint64_t>(st.hi));
  if (a.mode == ORC_LUT_EQUALIZE) out.params.set("cdf_min", st.cdf_min);
}

int g_threads = 0;

void add_oracle_tasks(task::TaskRegistry& r) {
  r.add({.flag = "LUT_GEN",
         .required_params = {"rows", "cols"},
         .payload_rule = [](const wire::ParamMap& p) {
           const LutArgs a = lut_args(p, true);
           return a.rows * a.cols * 2;
         },
         .handler = [](const wire::ParamMap& p, std::span<const std::uint8_t> in) {
           const LutArgs a = lut_args(p, true);
           task::TaskOutput out;
           out.payload.resize(kLutBytes);
           orc_lut_stats st{};
           orc_lut_gen(reinterpret_cast<const std::uint16_t*>(in.data()), a.rows * a.cols, a.mode,
                       reinterpret_cast<std::uint16_t*>(out.payload.data()), &st, g_threads);
           lut_result(out, a, st);
           return out;
         }});
  r.add({.flag = "LUT_APPLY",
         .required_params = {"rows", "cols"},
         .payload_rule = [](const wire::ParamMap& p) {
           const LutArgs a = lut_args(p, false);
           return capped(kLutBytes, a.rows * a.cols * 2);
         },
         .handler = [](const wire::ParamMap& p, std::span<const std::uint8_t> in) {
           const LutArgs a = lut_args(p, false);
           task::TaskOutput out;
           out.payload.resize(a.rows * a.cols * 2);
           orc_lut_apply(reinterpret_cast<const std::uint16_t*>(in.data()),
                         reinterpret_cast<const std::uint16_t*>(in.data() + kLutBytes),
                         reinterpret_cast<std::uint16_t*>(out.payload.data()), a.rows * a.cols,
                         g_threads);
           out.params.set("rows", a.rows);
           out.params.set("cols", a.cols);
           return out;
         }});
  r.add({.flag = "LUT_CORRECT",
         .required_params = {"rows", "cols"},
         .payload_rule = [](const wire::ParamMap& p) {
           const LutArgs a = lut_args(p, true);
           return a.rows * a.cols * 2;
         },
         .handler = [](const wire::ParamMap& p, std::span<const std::uint8_t> in) {
           const LutArgs a = lut_args(p, true);
           task::TaskOutput out;
           out.payload.resize(a.rows * a.cols * 2);
           std::vector<std::uint16_t> lut(65536);
           orc_lut_stats st{};
           orc_lut_correct(reinterpret_cast<const std::uint16_t*>(in.data()),
                           reinterpret_cast<std::uint16_t*>(out.payload.data()), a.rows * a.cols,
                           a.mode, lut.data(), &st, g_threads);
           lut_result(out, a, st);
           return out;
         }});
  r.add({.flag = "MATMUL",
         .required_params = {"m", "k", "n"},
         .payload_rule = [](const wire::ParamMap& p) {
           const MatArgs a = mat_args(p);
           return (a.m * a.k + a.k * a.n) * 4;
         },
         .handler = [](const wire::ParamMap& p, std::span<const std::uint8_t> in) {
           const MatArgs a = mat_args(p);
           std::vector<float> A(a.m * a.k), B(a.k * a.n);
           std::memcpy(A.data(), in.data(), A.size() * 4);
           std::memcpy(B.data(), in.data() + A.size() * 4, B.size() * 4);
           orc_round_matrix(a.prec, A.data(), A.data(), A.size(), g_threads);
           orc_round_matrix(a.prec, B.data(), B.data(), B.size(), g_threads);
           task::TaskOutput out;
           out.payload.resize(a.m * a.n * 4);
           orc_matmul_f32(a.m, a.n, a.k, A.data(), B.data(),
                          reinterpret_cast<float*>(out.payload.data()), g_threads);
           out.params.set("m", a.m);
           out.params.set("n", a.n);
           out.params.set("k", a.k);
           out.params.set("prec", a.prec == ORC_PREC_TF32 ? "tf32"
                                  : a.prec == ORC_PREC_BF16 ? "bf16" : "f32");
           return out;
         }});
}

std::shared_ptr<const task::DeviceList> test_devices() {
  devinfo::DeviceInfo d;
  d.name = "Test Device";
  d.compute_capability = "1.3";
  d.warp_size = 32;
  d.clock_rate_khz = 1300000;
  d.multi_processor_count = 30;
  d.total_global_memory = 4294967296ull;
  auto list = std::make_shared<task::DeviceList>();
  list->push_back(d);
  return list;
}

// Builtins (fixed test device, as the reference tests do) + oracle tasks.
const task::TaskRegistry& registry() {
  static const task::TaskRegistry* r = [] {
    auto* reg = new task::TaskRegistry(task::make_builtin_registry(par::ExecPlan{}, test_devices()));
    add_oracle_tasks(*reg);
    return reg;
  }();
  return *r;
}

struct ServerHandle {
  std::unique_ptr<srv::Server> server;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_set_threads(int threads) { g_threads = threads; }

int ref_encode_header(const char* flag, int marker, const char* params, const char* name,
                      std::uint8_t* out) {
  return guarded([&] {
    wire::TaskHeader h{flag, static_cast<std::uint8_t>(marker), params, name};
    const wire::HeaderBytes b = wire::encode_header(h);
    std::memcpy(out, b.data(), b.size());
  });
}

int ref_decode_header(const std::uint8_t* in, std::size_t len, char* flag, int* marker,
                      char* params, char* name) {
  return guarded([&] {
    const wire::TaskHeader h = wire::decode_header(std::span<const std::uint8_t>(in, len));
    put(h.task_flag, flag, 64);
    *marker = h.data_marker;
    put(h.params, params, 256);
    put(h.output_name, name, 64);
  });
}

// parse then serialize (the ParamMap round trip), plus get_uint(key) if key.
int ref_params_roundtrip(const char* text, char* out, std::size_t cap) {
  return guarded([&] { put(wire::ParamMap::parse(text).serialize(), out, cap); });
}

int ref_params_get_uint(const char* text, const char* key, std::uint64_t* value) {
  return guarded([&] { *value = wire::ParamMap::parse(text).get_uint(key); });
}

int ref_expected_payload_len(const char* flag, const char* params, std::uint64_t* len) {
  return guarded([&] {
    const task::TaskDescriptor& d = registry().lookup(flag);
    *len = d.payload_rule(wire::ParamMap::parse(params));
  });
}

int ref_sanitize_message(const char* text, const char* existing, char* out, std::size_t cap) {
  return guarded([&] { put(task::sanitize_message(text, wire::ParamMap::parse(existing)), out, cap); });
}

// srv::handle_connection over a MemoryStream; response frame bytes out.
int ref_handle_request(const std::uint8_t* req, std::size_t len, std::uint8_t* resp,
                       std::size_t cap, std::size_t* resp_len) {
  return guarded([&] {
    wire::MemoryStream stream(std::vector<std::uint8_t>(req, req + len));
    srv::handle_connection(stream, registry());
    const auto& w = stream.written();
    *resp_len = w.size();
    if (w.size() > cap) fail(Errc::SizeMismatch, "response buffer too small");
    std::memcpy(resp, w.data(), w.size());
  });
}

int ref_server_start(int port, int max_tasks, void** handle, std::uint16_t* bound) {
  return guarded([&] {
    auto h = std::make_unique<ServerHandle>();
    srv::ServerConfig cfg;
    cfg.bind_addr = "127.0.0.1";
    cfg.port = static_cast<std::uint16_t>(port);
    cfg.max_tasks = max_tasks;
    h->server = std::make_unique<srv::Server>(cfg, registry());
    h->server->start();
    *bound = h->server->port();
    *handle = h.release();
  });
}

int ref_server_stop(void* handle) {
  return guarded([&] {
    auto* h = static_cast<ServerHandle*>(handle);
    h->server->stop();
    delete h;
  });
}

// client::submit; response payload copied to resp (cap bytes).
int ref_submit(const char* host, int port, const char* flag, const char* params,
               const std::uint8_t* payload, std::size_t len, const char* name, std::uint8_t* resp,
               std::size_t cap, std::size_t* resp_len, char* status, char* resp_params,
               char* resp_name) {
  return guarded([&] {
    const client::TaskResult r = client::submit(host, static_cast<std::uint16_t>(port), flag,
                                              wire::ParamMap::parse(params),
                                              std::span<const std::uint8_t>(payload, len), name);
    put(r.status, status, 64);
    put(r.params.serialize(), resp_params, 256);
    put(r.output_name, resp_name, 64);
    *resp_len = r.payload.size();
    if (r.payload.size() > cap) fail(Errc::SizeMismatch, "response buffer too small");
    if (!r.payload.empty()) std::memcpy(resp, r.payload.data(), r.payload.size());
  });
}

// The reference's DEVINFO XML for records given in include/gpcx.h's layout.
int ref_devinfo_render(const gpcx_device_info* devs, int n, char* out, std::size_t cap,
                       std::size_t* len) {
  return guarded([&] {
    std::vector<devinfo::DeviceInfo> list;
    for (int i = 0; i < n; ++i) {
      const gpcx_device_info& s = devs[i];
      devinfo::DeviceInfo d;
      d.name = std::string(s.name, strnlen(s.name, sizeof(s.name)));
      d.compute_capability =
          std::string(s.compute_capability, strnlen(s.compute_capability, sizeof(s.compute_capability)));
      d.warp_size = s.warp_size;
      d.total_constant_memory = s.total_constant_memory;
      d.total_global_memory = s.total_global_memory;
      d.shared_memory_per_block = s.shared_memory_per_block;
      d.clock_rate_khz = s.clock_rate_khz;
      d.multi_processor_count = s.multi_processor_count;
      d.registers_per_block = s.registers_per_block;
      d.max_threads_per_block = s.max_threads_per_block;
      for (int j = 0; j < 3; ++j) {
        d.max_grid_size[j] = s.max_grid_size[j];
        d.max_threads_dim[j] = s.max_threads_dim[j];
      }
      list.push_back(d);
    }
    const std::string xml = devinfo::to_xml(list);
    *len = xml.size();
    put(xml, out, cap);
  });
}

// Reference demosaic kernels (gradient=0/1) and the independent gpcref oracle.
int ref_demosaic(int gradient, int use_gpcref, const char* phase, std::size_t rows,
                 std::size_t cols, const std::uint16_t* in, std::uint16_t* rgb, int workers) {
  return guarded([&] {
    img::BayerImage image;
    image.rows = rows;
    image.cols = cols;
    image.phase = img::phase_from_string(phase);
    image.samples.assign(in, in + rows * cols);
    img::RgbImage out;
    if (use_gpcref) {
      out = gradient ? gpcref::demosaic_gradient_ref(image) : gpcref::demosaic_bilinear_ref(image);
    } else {
      par::ExecPlan plan;
      if (workers > 0) plan.workers = workers;
      out = gradient ? img::demosaic_gradient(image, plan) : img::demosaic_bilinear(image, plan);
    }
    const std::size_t n = rows * cols;
    std::memcpy(rgb, out.r.data(), n * 2);
    std::memcpy(rgb + n, out.g.data(), n * 2);
    std::memcpy(rgb + 2 * n, out.b.data(), n * 2);
  });
}

// The reference's normal equations for a polynomial fit of `order`:
// A = V^T V ((order+1)^2 Hankel matrix of power sums, row-major) and
// b = V^T y with V[i][j] = xs[i]^j -- two contractions the reference itself
// computes (gpc::lsq::build_normal_system, proj/src/lsq.cpp:69-90), used to
// anchor the MATMUL oracle and the B200 MATMUL on reference-computed values.
int ref_normal_system(const double* xs, const double* ys, std::size_t n, int order,
                      double* a_out, double* b_out) {
  return guarded([&] {
    const lsq::NormalSystem sys = lsq::build_normal_system(
        std::span<const double>(xs, n), std::span<const double>(ys, n), order, par::ExecPlan{});
    std::memcpy(a_out, sys.a.a.data(), sys.a.a.size() * sizeof(double));
    std::memcpy(b_out, sys.b.data(), sys.b.size() * sizeof(double));
  });
}

}  // extern "C"
