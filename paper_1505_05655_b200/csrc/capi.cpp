// capi.cpp -- the extern "C" surface of include/gpcx.h.  Every entry point
// converts C++ failures into a gpcx_status (1 + Errc ordinal) and a
// thread-local message; nothing throws across the boundary.
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/gpcx.h"
#include "cuda_util.hpp"
#include "host/devinfo.hpp"
#include "host/executor.hpp"
#include "host/tcp.hpp"
#include "host/peer.hpp"
#include "host/registry.hpp"
#include "host/runtime.hpp"
#include "host/server.hpp"
#include "host/task_spec.hpp"
#include "kernels.hpp"

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& body) {
  try {
    body();
    g_last_error.clear();
    return GPCX_OK;
  } catch (const gpcx::Error& e) {
    g_last_error = e.what();
    return gpcx::to_status(e.code());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return gpcx::to_status(gpcx::Errc::TaskFailed);
  } catch (...) {
    g_last_error = "unknown failure";
    return gpcx::to_status(gpcx::Errc::TaskFailed);
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

void copy_text(const std::string& text, char* out, uint64_t cap) {
  if (out == nullptr || cap == 0) {
    if (!text.empty()) gpcx::fail(gpcx::Errc::SizeMismatch, "text buffer too small");
    return;
  }
  if (text.size() + 1 > cap)
    gpcx::fail(gpcx::Errc::SizeMismatch, "text buffer holds " + std::to_string(cap) +
                                             " bytes, need " + std::to_string(text.size() + 1));
  std::memcpy(out, text.c_str(), text.size() + 1);
}

const char* nz(const char* s) { return s != nullptr ? s : ""; }

void need_ws(void* ws, uint64_t have, uint64_t want) {
  if (want > 0 && (ws == nullptr || have < want))
    gpcx::fail(gpcx::Errc::SizeMismatch, "workspace holds " + std::to_string(have) +
                                             " bytes, need " + std::to_string(want));
}

void need_u32(uint64_t n) {
  if (n >= (1ull << 32)) gpcx::fail(gpcx::Errc::TooLarge, "more than 2^32-1 samples per call");
}

}  // namespace

extern "C" {

int gpcx_abi_version(void) { return GPCX_ABI_VERSION; }

int gpcx_init(int ndev, const int* devices) {
  return guarded([&] {
    std::vector<int> devs;
    if (ndev < 0) gpcx::fail(gpcx::Errc::BadValue, "negative device count");
    for (int i = 0; i < ndev; ++i) devs.push_back(devices != nullptr ? devices[i] : i);
    gpcx::rt::Runtime::get().init(devs);
  });
}

int gpcx_shutdown(void) {
  return guarded([] {
    gpcx::rt::Runtime::get().shutdown();
    gpcx::rt::pinned_trim();
  });
}

int gpcx_device_count(int* count) {
  return guarded([&] { *count = gpcx::rt::Runtime::get().ndev(); });
}

int gpcx_device_health(int index, int* healthy, char* why, uint64_t why_cap) {
  return guarded([&] {
    gpcx::rt::Runtime& R = gpcx::rt::Runtime::get();
    if (index < 0 || index >= R.ndev()) gpcx::fail(gpcx::Errc::BadValue, "device index");
    if (healthy != nullptr) *healthy = R.healthy(index) ? 1 : 0;
    copy_text(R.health_reason(index), why, why_cap);
  });
}

int gpcx_debug_fault(int index, int kind) {
  return guarded([&] {
    gpcx::rt::Runtime& R = gpcx::rt::Runtime::get();
    if (index < 0 || index >= R.ndev()) gpcx::fail(gpcx::Errc::BadValue, "device index");
    if (kind == 0) {
      R.quarantine_index(index, "gpcx_debug_fault");
      return;
    }
    if (kind != 1) gpcx::fail(gpcx::Errc::BadValue, "fault kind");
    gpcx::rt::SlotLease s = R.acquire(index);
    gpcx::synth::launch_trap(s->stream);
    GPCX_CUDA(cudaStreamSynchronize(s->stream));  // fails: the trap is sticky
  });
}

const char* gpcx_last_error(void) { return g_last_error.c_str(); }

const char* gpcx_status_name(int status) {
  if (status == GPCX_OK) return "OK";
  if (status < 1 || status > gpcx::kErrcCount) return "Unknown";
  return gpcx::errc_name(static_cast<gpcx::Errc>(status - 1));
}

const char* gpcx_response_code(int status) {
  static thread_local std::string code;
  if (status == GPCX_OK) return "OK";
  if (status < 1 || status > gpcx::kErrcCount) return "TASK_FAILED";
  code = gpcx::response_code(static_cast<gpcx::Errc>(status - 1));
  return code.c_str();
}

int gpcx_payload_len(const char* flag, const char* params, uint64_t* len) {
  return guarded([&] {
    const auto f = gpcx::task::flag_of(nz(flag));
    *len = gpcx::task::payload_len(f, gpcx::wire::ParamMap::parse(nz(params)));
  });
}

int gpcx_output_len(const char* flag, const char* params, uint64_t* len) {
  return guarded([&] {
    const auto f = gpcx::task::flag_of(nz(flag));
    const auto p = gpcx::wire::ParamMap::parse(nz(params));
    *len = f == gpcx::task::Flag::DevInfo ? gpcx::exec::devinfo_xml().size()
                                          : gpcx::task::output_len(f, p);
  });
}

int gpcx_required_params(const char* flag, char* out, uint64_t cap) {
  return guarded([&] {
    std::string text;
    for (const std::string& k : gpcx::task::required_params(gpcx::task::flag_of(nz(flag)))) {
      if (!text.empty()) text += ',';
      text += k;
    }
    copy_text(text, out, cap);
  });
}

int gpcx_flags(char* out, uint64_t cap) {
  return guarded([&] {
    std::string text;
    for (const auto f : gpcx::task::all_flags()) {
      if (!text.empty()) text += ',';
      text += gpcx::task::flag_name(f);
    }
    copy_text(text, out, cap);
  });
}

int gpcx_run(const char* flag, const char* params, const void* in, uint64_t in_len, void* out,
             uint64_t out_cap, uint64_t* out_len, char* result_params,
             uint64_t result_params_cap) {
  return guarded([&] {
    const auto f = gpcx::task::flag_of(nz(flag));
    const auto p = gpcx::wire::ParamMap::parse(nz(params));
    const uint64_t want = f == gpcx::task::Flag::DevInfo ? gpcx::exec::devinfo_xml().size()
                                                         : gpcx::task::output_len(f, p);
    if (out_cap < want)
      gpcx::fail(gpcx::Errc::SizeMismatch, "output buffer holds " + std::to_string(out_cap) +
                                               " bytes, need " + std::to_string(want));
    if (in_len > 0 && in == nullptr) gpcx::fail(gpcx::Errc::BadValue, "null payload");
    const auto result = gpcx::exec::execute(
        f, p, std::span<const std::uint8_t>(static_cast<const std::uint8_t*>(in), in_len),
        std::span<std::uint8_t>(static_cast<std::uint8_t*>(out), want));
    if (out_len != nullptr) *out_len = want;
    if (result_params != nullptr) copy_text(result.serialize(), result_params, result_params_cap);
  });
}

int gpcx_lut_host(int op, int mode, uint64_t rows, uint64_t cols, const uint16_t* img,
                  const uint16_t* lut_in, uint16_t* out, uint16_t* lut_out,
                  gpcx_lut_stats* stats) {
  return guarded([&] {
    using gpcx::task::Flag;
    const Flag f = op == GPCX_OP_LUT_GEN     ? Flag::LutGen
                   : op == GPCX_OP_LUT_APPLY ? Flag::LutApply
                   : op == GPCX_OP_LUT_CORRECT
                       ? Flag::LutCorrect
                       : (gpcx::fail(gpcx::Errc::BadValue, "op " + std::to_string(op)), Flag::LutGen);
    if (rows == 0 || cols == 0) gpcx::fail(gpcx::Errc::BadValue, "rows and cols must be positive");
    if (mode != GPCX_LUT_EQUALIZE && mode != GPCX_LUT_STRETCH)
      gpcx::fail(gpcx::Errc::BadValue, "mode " + std::to_string(mode));
    if (img == nullptr || out == nullptr || (f == Flag::LutApply && lut_in == nullptr))
      gpcx::fail(gpcx::Errc::BadValue, "null buffer");
    need_u32(rows * cols);
    gpcx::task::LutParams p;
    p.rows = rows;
    p.cols = cols;
    p.mode = mode;
    const gpcx_lut_stats st = gpcx::exec::lut_host(f, p, img, lut_in, out, lut_out);
    if (stats != nullptr) *stats = st;
  });
}

int gpcx_matmul_host(int prec, uint64_t m, uint64_t n, uint64_t k, const float* A,
                     const float* B, float* C) {
  return guarded([&] {
    if (m == 0 || n == 0 || k == 0) gpcx::fail(gpcx::Errc::BadValue, "dimensions must be positive");
    if (prec != GPCX_PREC_F32 && prec != GPCX_PREC_TF32 && prec != GPCX_PREC_BF16)
      gpcx::fail(gpcx::Errc::BadValue, "prec " + std::to_string(prec));
    gpcx::task::MatmulParams p;
    p.m = m;
    p.n = n;
    p.k = k;
    p.prec = prec;
    gpcx::exec::matmul_host(p, A, B, C);
  });
}

void* gpcx_pinned_alloc(uint64_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes == 0 ? 1 : bytes) != cudaSuccess) {
    cudaGetLastError();
    g_last_error = "cudaMallocHost failed";
    return nullptr;
  }
  return p;
}

void gpcx_pinned_free(void* ptr) {
  if (ptr != nullptr) cudaFreeHost(ptr);
}

int gpcx_lut_workspace_size(uint64_t n, uint64_t* bytes) {
  return guarded([&] {
    need_u32(n);
    *bytes = gpcx::lut::workspace_bytes(n);
  });
}

int gpcx_lut_hist_device(const uint16_t* img, uint64_t n, uint32_t* hist, void* ws,
                         uint64_t ws_bytes, void* stream) {
  return guarded([&] {
    need_u32(n);
    need_ws(ws, ws_bytes, gpcx::lut::workspace_bytes());
    gpcx::lut::launch_hist(img, n, hist, ws, as_stream(stream));
  });
}

int gpcx_lut_from_hist_device(const uint32_t* hist, int mode, uint16_t* lut,
                              gpcx_lut_stats* stats, void* ws, uint64_t ws_bytes,
                              void* stream) {
  return guarded([&] {
    if (mode != GPCX_LUT_EQUALIZE && mode != GPCX_LUT_STRETCH)
      gpcx::fail(gpcx::Errc::BadValue, "mode " + std::to_string(mode));
    need_ws(ws, ws_bytes, gpcx::lut::workspace_bytes());
    gpcx::lut::launch_from_hist(hist, mode, lut, stats, ws, as_stream(stream));
  });
}

int gpcx_lut_correct_from_hist_device(const uint32_t* hist, int mode, const uint16_t* in,
                                      uint16_t* out, uint64_t n, uint16_t* lut,
                                      gpcx_lut_stats* stats, void* ws, uint64_t ws_bytes,
                                      void* stream) {
  return guarded([&] {
    if (mode != GPCX_LUT_EQUALIZE && mode != GPCX_LUT_STRETCH)
      gpcx::fail(gpcx::Errc::BadValue, "mode " + std::to_string(mode));
    need_u32(n);
    need_ws(ws, ws_bytes, gpcx::lut::workspace_bytes());
    gpcx::lut::launch_correct_from_hist(hist, mode, in, out, n, lut, stats, ws,
                                        as_stream(stream));
  });
}

int gpcx_lut_minmax_device(const uint16_t* img, uint64_t n, gpcx_lut_stats* stats, void* ws,
                           uint64_t ws_bytes, void* stream) {
  return guarded([&] {
    need_u32(n);
    need_ws(ws, ws_bytes, gpcx::lut::workspace_bytes());
    gpcx::lut::launch_minmax(img, n, stats, ws, as_stream(stream));
  });
}

int gpcx_lut_from_minmax_device(const gpcx_lut_stats* stats, uint16_t* lut, void* stream) {
  return guarded([&] { gpcx::lut::launch_from_minmax(stats, lut, as_stream(stream)); });
}

int gpcx_lut_gen_device(const uint16_t* img, uint64_t n, int mode, uint16_t* lut,
                        gpcx_lut_stats* stats, void* ws, uint64_t ws_bytes, void* stream) {
  return guarded([&] {
    need_u32(n);
    need_ws(ws, ws_bytes, gpcx::lut::workspace_bytes());
    const cudaStream_t s = as_stream(stream);
    if (mode == GPCX_LUT_EQUALIZE) {
      gpcx::lut::launch_hist_lut(img, n, mode, lut, stats, ws, s);
    } else if (mode == GPCX_LUT_STRETCH) {
      gpcx::lut::launch_minmax(img, n, stats, ws, s);
      gpcx::lut::launch_from_minmax(stats, lut, s);
    } else {
      gpcx::fail(gpcx::Errc::BadValue, "mode " + std::to_string(mode));
    }
  });
}

int gpcx_lut_apply_device(const uint16_t* lut, const uint16_t* in, uint16_t* out, uint64_t n,
                          void* stream) {
  return guarded([&] { gpcx::lut::launch_apply(lut, in, out, n, as_stream(stream)); });
}

int gpcx_lut_correct_device(const uint16_t* in, uint16_t* out, uint64_t n, int mode,
                            uint16_t* lut, gpcx_lut_stats* stats, void* ws, uint64_t ws_bytes,
                            void* stream) {
  return guarded([&] {
    need_u32(n);
    need_ws(ws, ws_bytes, gpcx::lut::workspace_bytes());
    if (mode != GPCX_LUT_EQUALIZE && mode != GPCX_LUT_STRETCH)
      gpcx::fail(gpcx::Errc::BadValue, "mode " + std::to_string(mode));
    gpcx::lut::launch_correct(in, out, n, mode, lut, stats, ws, as_stream(stream), ws_bytes);
  });
}

static_assert(sizeof(cudaIpcMemHandle_t) == GPCX_IPC_HANDLE_BYTES, "IPC handle size");

struct gpcx_lut_peer {
  gpcx::peer::LutRank rank;
  gpcx_lut_peer(int r, int n) : rank(r, n) {}
};

int gpcx_lut_peer_create(int rank, int nranks, gpcx_lut_peer** out) {
  return guarded([&] {
    if (out == nullptr) gpcx::fail(gpcx::Errc::BadValue, "null output");
    *out = new gpcx_lut_peer(rank, nranks);
  });
}

int gpcx_lut_peer_ipc_handle(const gpcx_lut_peer* p, void* handle) {
  return guarded([&] {
    if (p == nullptr || handle == nullptr) gpcx::fail(gpcx::Errc::BadValue, "null argument");
    const cudaIpcMemHandle_t h = p->rank.handle();
    std::memcpy(handle, &h, sizeof(h));
  });
}

int gpcx_lut_peer_connect(gpcx_lut_peer* p, const void* handles) {
  return guarded([&] {
    if (p == nullptr || handles == nullptr) gpcx::fail(gpcx::Errc::BadValue, "null argument");
    std::vector<cudaIpcMemHandle_t> hs(p->rank.nranks());
    std::memcpy(hs.data(), handles, hs.size() * sizeof(cudaIpcMemHandle_t));
    p->rank.connect(hs.data());
  });
}

int gpcx_lut_peer_destroy(gpcx_lut_peer* p) {
  return guarded([&] { delete p; });
}

int gpcx_lut_correct_peer_device(gpcx_lut_peer* p, const uint16_t* in, uint16_t* out,
                                 uint64_t n, int mode, uint16_t* lut, gpcx_lut_stats* stats,
                                 void* ws, uint64_t ws_bytes, void* stream) {
  return guarded([&] {
    if (p == nullptr) gpcx::fail(gpcx::Errc::BadValue, "null peer group");
    if (mode != GPCX_LUT_EQUALIZE && mode != GPCX_LUT_STRETCH)
      gpcx::fail(gpcx::Errc::BadValue, "mode " + std::to_string(mode));
    need_u32(n);
    need_ws(ws, ws_bytes, gpcx::lut::workspace_bytes());
    p->rank.correct(in, out, n, mode, lut, stats, ws, as_stream(stream), ws_bytes);
  });
}

int gpcx_matmul_workspace_size(int prec, uint64_t m, uint64_t n, uint64_t k, uint64_t* bytes) {
  return guarded([&] {
    *bytes = prec == GPCX_PREC_F32 ? gpcx::gemm::sgemm_workspace_bytes(m, n, k)
                                   : gpcx::gemm::tc_workspace_bytes(prec, m, n, k);
  });
}

int gpcx_matmul_device(int prec, uint64_t m, uint64_t n, uint64_t k, const float* A,
                       uint64_t lda, const float* B, uint64_t ldb, float* C, uint64_t ldc,
                       void* ws, uint64_t ws_bytes, void* stream) {
  return guarded([&] {
    if (lda < k || ldb < n || ldc < n)
      gpcx::fail(gpcx::Errc::BadValue, "leading dimension smaller than the row length");
    if (prec == GPCX_PREC_F32) {
      // the workspace is optional here (same bits either way, A^T path faster)
      gpcx::gemm::launch_sgemm(m, n, k, A, lda, B, ldb, C, ldc, ws, ws_bytes, as_stream(stream));
    } else if (prec == GPCX_PREC_TF32 || prec == GPCX_PREC_BF16) {
      need_ws(ws, ws_bytes, gpcx::gemm::tc_workspace_bytes(prec, m, n, k));
      gpcx::gemm::launch_tc(prec, m, n, k, A, lda, B, ldb, C, ldc, ws, as_stream(stream));
    } else {
      gpcx::fail(gpcx::Errc::BadValue, "prec " + std::to_string(prec));
    }
  });
}

int gpcx_synth_image_device(int kind, uint64_t seed, uint64_t rows, uint64_t cols, uint64_t row0,
                            uint64_t nrows, uint16_t* out, void* stream) {
  return guarded([&] {
    if (kind != GPCX_IMG_RAMP12 && kind != GPCX_IMG_UNIFORM16)
      gpcx::fail(gpcx::Errc::BadValue, "image kind " + std::to_string(kind));
    gpcx::synth::launch_image(kind, seed, rows, cols, row0, nrows, out, as_stream(stream));
  });
}

int gpcx_synth_matrix_device(int kind, uint64_t seed, uint64_t rows, uint64_t cols,
                             uint64_t row0, uint64_t nrows, float* out, void* stream) {
  return guarded([&] {
    if (kind != GPCX_MAT_EXACT8 && kind != GPCX_MAT_UNIFORM32)
      gpcx::fail(gpcx::Errc::BadValue, "matrix kind " + std::to_string(kind));
    gpcx::synth::launch_matrix(kind, seed, rows, cols, row0, nrows, out, as_stream(stream));
  });
}

int gpcx_demosaic_device(int gradient, int phase, const uint16_t* in, uint16_t* out,
                         uint64_t rows, uint64_t cols, void* stream) {
  return guarded([&] {
    if (phase < 0 || phase > 3) gpcx::fail(gpcx::Errc::BadValue, "phase " + std::to_string(phase));
    gpcx::demosaic::launch(gradient != 0, phase, in, out, rows, cols, as_stream(stream));
  });
}

int gpcx_devinfo_probe(gpcx_device_info* out, int cap, int* count) {
  return guarded([&] {
    const auto list = gpcx::devinfo::probe_cuda(gpcx::rt::Runtime::get().devices());
    *count = static_cast<int>(list.size());
    for (int i = 0; i < static_cast<int>(list.size()) && i < cap; ++i) {
      const auto& d = list[static_cast<std::size_t>(i)];
      gpcx_device_info& o = out[i];
      std::memset(&o, 0, sizeof(o));
      std::strncpy(o.name, d.name.c_str(), sizeof(o.name) - 1);
      std::strncpy(o.compute_capability, d.compute_capability.c_str(), sizeof(o.compute_capability) - 1);
      o.warp_size = d.warp_size;
      o.total_constant_memory = d.total_constant_memory;
      o.total_global_memory = d.total_global_memory;
      o.shared_memory_per_block = d.shared_memory_per_block;
      o.clock_rate_khz = d.clock_rate_khz;
      o.multi_processor_count = d.multi_processor_count;
      o.registers_per_block = d.registers_per_block;
      o.max_threads_per_block = d.max_threads_per_block;
      for (int j = 0; j < 3; ++j) {
        o.max_grid_size[j] = d.max_grid_size[static_cast<std::size_t>(j)];
        o.max_threads_dim[j] = d.max_threads_dim[static_cast<std::size_t>(j)];
      }
    }
  });
}

int gpcx_devinfo_render(const gpcx_device_info* devs, int n, char* out, uint64_t cap,
                        uint64_t* len) {
  return guarded([&] {
    std::vector<gpcx::devinfo::DeviceInfo> list;
    for (int i = 0; i < n; ++i) {
      const gpcx_device_info& s = devs[i];
      gpcx::devinfo::DeviceInfo d;
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
        d.max_grid_size[static_cast<std::size_t>(j)] = s.max_grid_size[j];
        d.max_threads_dim[static_cast<std::size_t>(j)] = s.max_threads_dim[j];
      }
      list.push_back(std::move(d));
    }
    const std::string xml = gpcx::devinfo::to_xml(list);
    if (len != nullptr) *len = xml.size();
    copy_text(xml, out, cap);
  });
}

int gpcx_digest_u16_device(const uint16_t* v, uint64_t n, uint64_t index0, uint64_t* digest,
                           void* stream) {
  return guarded([&] { gpcx::synth::launch_digest(v, n, index0, digest, as_stream(stream)); });
}

struct gpcx_server_handle {
  gpcx::task::TaskRegistry registry;
  std::unique_ptr<gpcx::srv::Server> server;
};

int gpcx_server_start(const char* bind_addr, uint16_t port, int max_tasks, int idle_timeout_ms,
                      void** handle, uint16_t* bound_port) {
  return guarded([&] {
    auto h = std::make_unique<gpcx_server_handle>();
    h->registry = gpcx::task::make_b200_registry();
    gpcx::srv::ServerConfig cfg;
    cfg.bind_addr = bind_addr != nullptr ? bind_addr : "0.0.0.0";
    cfg.port = port;
    cfg.max_tasks = max_tasks;
    if (idle_timeout_ms > 0) cfg.idle_timeout = std::chrono::milliseconds(idle_timeout_ms);
    const char* quiet = std::getenv("GPCX_QUIET");
    cfg.log = !(quiet != nullptr && quiet[0] == '1');
    h->server = std::make_unique<gpcx::srv::Server>(cfg, h->registry);
    h->server->start();
    if (bound_port != nullptr) *bound_port = h->server->port();
    *handle = h.release();
  });
}

int gpcx_server_stop(void* handle) {
  return guarded([&] {
    auto* h = static_cast<gpcx_server_handle*>(handle);
    if (h == nullptr) return;
    h->server->stop();
    delete h;
  });
}

int gpcx_server_stats_get(void* handle, gpcx_server_stats* out) {
  return guarded([&] {
    auto* h = static_cast<gpcx_server_handle*>(handle);
    if (h == nullptr || out == nullptr) gpcx::fail(gpcx::Errc::BadValue, "null argument");
    const gpcx::srv::ServerStats st = h->server->stats();
    *out = gpcx_server_stats{st.requests, st.recv_ms, st.task_ms, st.send_ms, st.busy, st.dropped};
  });
}

int gpcx_handle_request(const uint8_t* req, uint64_t req_len, uint8_t* resp, uint64_t resp_cap,
                        uint64_t* resp_len) {
  return guarded([&] {
    static const gpcx::task::TaskRegistry* registry =
        new gpcx::task::TaskRegistry(gpcx::task::make_b200_registry());
    gpcx::wire::MemoryStream stream(std::vector<std::uint8_t>(req, req + req_len));
    gpcx::srv::serve_stream(stream, *registry);
    const auto& bytes = stream.written();
    if (resp_len != nullptr) *resp_len = bytes.size();
    if (bytes.size() > resp_cap)
      gpcx::fail(gpcx::Errc::SizeMismatch, "response buffer holds " + std::to_string(resp_cap) +
                                               " bytes, need " + std::to_string(bytes.size()));
    if (!bytes.empty()) std::memcpy(resp, bytes.data(), bytes.size());
  });
}

int gpcx_client_submit(const char* host, uint16_t port, const char* flag, const char* params,
                       const void* const* parts, const uint64_t* part_len, int nparts,
                       const char* output_name, void* resp, uint64_t resp_cap,
                       uint64_t* resp_len, char* status, uint64_t status_cap,
                       char* resp_params, uint64_t resp_params_cap) {
  return guarded([&] {
    std::uint64_t total = 0;
    for (int i = 0; i < nparts; ++i) total += part_len[i];
    gpcx::wire::TaskHeader h;
    h.task_flag = nz(flag);
    h.params = gpcx::wire::ParamMap::parse(nz(params)).serialize();
    h.output_name = nz(output_name);
    h.data_marker = total > 0 ? gpcx::wire::kMarkerData : gpcx::wire::kMarkerNone;
    if (total > gpcx::wire::kMaxPayload) gpcx::fail(gpcx::Errc::TooLarge, "payload over the cap");
    const gpcx::wire::HeaderBytes raw = gpcx::wire::encode_header(h);
    gpcx::tcp::Conn s = gpcx::tcp::dial(nz(host), port);
    s.write_all(raw);
    for (int i = 0; i < nparts; ++i)
      if (part_len[i] > 0)
        s.write_all(std::span<const std::uint8_t>(static_cast<const std::uint8_t*>(parts[i]), part_len[i]));
    gpcx::wire::HeaderBytes rh;
    gpcx::wire::read_exact(s, rh);
    const gpcx::wire::TaskHeader r = gpcx::wire::decode_header(rh);
    const std::uint64_t n = gpcx::wire::response_payload_len(r);
    if (resp_len != nullptr) *resp_len = n;
    if (n > resp_cap)
      gpcx::fail(gpcx::Errc::SizeMismatch, "response payload is " + std::to_string(n) +
                                               " bytes, buffer holds " + std::to_string(resp_cap));
    if (n > 0) gpcx::wire::read_exact(s, std::span<std::uint8_t>(static_cast<std::uint8_t*>(resp), n));
    copy_text(r.task_flag, status, status_cap);
    copy_text(r.params, resp_params, resp_params_cap);
  });
}

}  // extern "C"
