/*
 * gpcx.h -- C ABI of the B200-native task backend (libgpcx.so).
 *
 * This is the drop-in boundary between the reference `gpc` server's task
 * plugin contract and the sm_100a kernels.  The reference registers tasks as
 *
 *   struct TaskDescriptor { std::string flag;
 *                           std::vector<std::string> required_params;
 *                           PayloadRule payload_rule;   // ParamMap -> u64
 *                           Handler handler; };         // (ParamMap, span) -> TaskOutput
 *   (/root/reference/proj/include/gpc/registry.hpp:23-37)
 *
 * and calls payload_rule before the payload is read (proj/src/server.cpp:73-93)
 * and handler from dispatch (proj/src/registry.cpp:79-120).  A reference-side
 * shim (integration/gpc_b200_tasks.cpp, shown in INTEGRATION.md) binds
 *
 *   payload_rule  -> gpcx_payload_len      handler -> gpcx_output_len + gpcx_run
 *
 * so the reference server serves LUT_GEN / LUT_APPLY / LUT_CORRECT / MATMUL
 * on the GPU without any C++ type crossing this boundary: only plain
 * pointers, sizes and NUL-terminated ASCII strings.  `params` strings use the
 * wire's own k=v,k=v text (proj/include/gpc/wire.hpp:55-62, the ';'->',' fold
 * included), so a shim passes header.params through unchanged.
 *
 * Errors.  Every entry point returns a gpcx_status: 0 = OK, otherwise
 * 1 + the ordinal of the reference's gpc::Errc enumerator
 * (proj/include/gpc/error.hpp:11-46), so a shim rethrows
 * `gpc::Error(static_cast<gpc::Errc>(rc - 1), gpcx_last_error())` and the
 * reference's response_code() mapping (proj/src/registry.cpp:38-60) yields
 * the identical ERR:<CODE>.  CUDA failures map to GPCX_E_TASK_FAILED
 * (-> ERR:TASK_FAILED); there is no CPU fallback -- without a usable GPU
 * every compute entry point fails with GPCX_E_TASK_FAILED.
 * gpcx_last_error() returns a thread-local message for the last failure on
 * the calling thread.
 *
 * Threading.  All entry points are reentrant.  gpcx_run may be called from
 * any number of executor threads at once (the reference runs up to
 * max_tasks handlers concurrently, proj/src/server.cpp:114-131); each call
 * takes its own stream and staging buffers from per-device pools.
 */
#ifndef GPCX_H
#define GPCX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2: gpcx_server_stats gained busy / dropped; health, debug-fault and synth= requests */
#define GPCX_ABI_VERSION 2

/* 0 = OK; n > 0 = 1 + gpc::Errc ordinal (proj/include/gpc/error.hpp:11-46). */
typedef enum gpcx_status {
  GPCX_OK = 0,
  GPCX_E_FIELD_TOO_LONG = 1,
  GPCX_E_INVALID_CHARACTER = 2,
  GPCX_E_BAD_MARKER = 3,
  GPCX_E_MALFORMED_PADDING = 4,
  GPCX_E_DUPLICATE_KEY = 5,
  GPCX_E_BAD_TOKEN = 6,
  GPCX_E_MISSING_PARAM = 7,
  GPCX_E_BAD_VALUE = 8,
  GPCX_E_OVERFLOW = 9,
  GPCX_E_TRUNCATED = 10,
  GPCX_E_PAYLOAD_MISMATCH = 11,
  GPCX_E_UNKNOWN_TASK = 12,
  GPCX_E_DUPLICATE_FLAG = 13,
  GPCX_E_TASK_FAILED = 14,
  GPCX_E_BAD_IMAGE = 15,
  GPCX_E_INSUFFICIENT_POINTS = 16,
  GPCX_E_SINGULAR = 17,
  GPCX_E_ORDER_TOO_HIGH = 18,
  GPCX_E_CONNECT_FAILED = 19,
  GPCX_E_BIND_FAILED = 20,
  GPCX_E_TIMED_OUT = 21,
  GPCX_E_IO_ERROR = 22,
  GPCX_E_UNSAFE_NAME = 23,
  GPCX_E_SIZE_MISMATCH = 24,
  GPCX_E_BAD_FORMAT = 25,
  GPCX_E_TOO_LARGE = 26,
  GPCX_E_SERVER_ERROR = 27
} gpcx_status;

/* LUT modes, synthetic generators and matmul precisions. */
enum { GPCX_LUT_EQUALIZE = 0, GPCX_LUT_STRETCH = 1 };
enum { GPCX_IMG_RAMP12 = 0, GPCX_IMG_UNIFORM16 = 1 };
enum { GPCX_MAT_EXACT8 = 0, GPCX_MAT_UNIFORM32 = 1 };
enum {
  GPCX_PREC_F32 = 0,  /* SIMT FP32, fp32 accumulate: reference precision     */
  GPCX_PREC_TF32 = 1, /* tcgen05 kind::tf32, inputs rounded RNA to tf32      */
  GPCX_PREC_BF16 = 2  /* tcgen05 kind::f16 (bf16), inputs rounded RNE to bf16 */
};

/* Device-resident LUT statistics (24 bytes). */
typedef struct gpcx_lut_stats {
  uint64_t n;       /* pixels counted                              */
  uint32_t lo, hi;  /* smallest / largest sample value present      */
  uint64_t cdf_min; /* equalize: histogram count at lo              */
} gpcx_lut_stats;

/* ------------------------------------------------------------------ */
/* Context                                                             */
/* ------------------------------------------------------------------ */

int gpcx_abi_version(void);
/* Bind the backend to `ndev` CUDA devices (ndev == 0: every visible one).
 * Idempotent for the same set.  gpcx_run shards across the bound devices
 * (row bands / block rows).  Implicitly called with ndev=0 by
 * the first gpcx_run if never called. */
int gpcx_init(int ndev, const int* devices);
int gpcx_shutdown(void);
int gpcx_device_count(int* count); /* devices bound (after init) */
/* Health of bound device `index` (0 .. count-1): *healthy = 1 while the
 * device takes work, 0 once quarantined after a sticky CUDA error (illegal
 * address, launch failure / trap, ...): no request is routed to it any
 * more and sharded requests use the remaining devices; with none left GPU
 * tasks answer ERR:TASK_FAILED.  `why` (may be NULL) receives the error
 * that caused the quarantine.  Rebinding with gpcx_init resets the state.
 * (The reference has no device state: its failure boundary is the handler
 * exception -> ERR:TASK_FAILED, proj/src/registry.cpp:113-118.) */
int gpcx_device_health(int index, int* healthy, char* why, uint64_t why_cap);
/* Test hook for the health machinery: kind 0 quarantines bound index
 * `index` without touching the GPU; kind 1 launches a kernel that traps on
 * that device (a real sticky error, surfacing as TASK_FAILED here and at
 * the device's next use).  Never called by the product paths. */
int gpcx_debug_fault(int index, int kind);
const char* gpcx_last_error(void);
/* gpc::errc_name(Errc) for a status (proj/src/error.cpp:5-36). */
const char* gpcx_status_name(int status);
/* The ERR:<CODE> suffix reference dispatch would send for a status
 * (proj/src/registry.cpp:38-60); "OK" for 0. */
const char* gpcx_response_code(int status);

/* ------------------------------------------------------------------ */
/* Task level: what a reference TaskDescriptor shim binds.              */
/* flag: task_flag slot text; params: params slot text (k=v,k=v).      */
/* ------------------------------------------------------------------ */

/* Replaces TaskDescriptor::payload_rule (registry.hpp:28) for the GPU
 * flags: payload bytes implied by the params, with the reference's
 * dim_product() rules (proj/src/wire.cpp:67-80): zero dim -> BAD_VALUE,
 * over the 1 GiB cap (wire.hpp:47) -> OVERFLOW (-> ERR:TOO_LARGE),
 * non-integer -> BAD_VALUE, absent -> MISSING_PARAM, unknown flag ->
 * UNKNOWN_TASK. */
int gpcx_payload_len(const char* flag, const char* params, uint64_t* len);
/* Response payload bytes the same request will produce. */
int gpcx_output_len(const char* flag, const char* params, uint64_t* len);
/* Required params of a flag, comma-separated (TaskDescriptor::required_params). */
int gpcx_required_params(const char* flag, char* out, uint64_t cap);
/* Flags this backend serves, comma-separated. */
int gpcx_flags(char* out, uint64_t cap);

/* Replaces TaskDescriptor::handler (registry.hpp:29-30).  `in` is the
 * request payload (host memory; pinned buffers from gpcx_pinned_alloc skip a
 * staging copy), `out` receives the response payload (out_cap >= the
 * gpcx_output_len value).  result_params receives the result params text
 * (without bytes=, which dispatch adds: registry.cpp:103-104). */
int gpcx_run(const char* flag, const char* params, const void* in,
             uint64_t in_len, void* out, uint64_t out_cap, uint64_t* out_len,
             char* result_params, uint64_t result_params_cap);

/* In-process host-buffer entry points without the wire's 1 GiB payload cap
 * (wire.hpp:47), for callers that hold a whole scene in memory (config C3:
 * a 32768^2 u16 image is 2 GiB).  Same planner, staging and kernels as
 * gpcx_run.  op: GPCX_OP_LUT_GEN (out = 65536-entry LUT), GPCX_OP_LUT_APPLY
 * (lut_in required), GPCX_OP_LUT_CORRECT (lut_out optional).  stats: host
 * pointer or NULL. */
enum { GPCX_OP_LUT_GEN = 0, GPCX_OP_LUT_APPLY = 1, GPCX_OP_LUT_CORRECT = 2 };
int gpcx_lut_host(int op, int mode, uint64_t rows, uint64_t cols,
                  const uint16_t* img, const uint16_t* lut_in, uint16_t* out,
                  uint16_t* lut_out, gpcx_lut_stats* stats);
/* C = A * B on host row-major f32 buffers (block rows across devices). */
int gpcx_matmul_host(int prec, uint64_t m, uint64_t n, uint64_t k,
                     const float* A, const float* B, float* C);

/* Page-locked host buffers for zero-staging requests/responses. */
void* gpcx_pinned_alloc(uint64_t bytes);
void gpcx_pinned_free(void* ptr);

/* ------------------------------------------------------------------ */
/* Device level: HBM-resident operands on a caller stream               */
/* (stream = cudaStream_t as void*; NULL = legacy default stream).      */
/* Used by the executor / planner and by bench.py's device-timed leg.   */
/* ------------------------------------------------------------------ */

/* Workspace (device bytes) recommended for a LUT call over n pixels.
 * Workspace must be zero-filled ONCE when allocated; the kernels leave it
 * zeroed again.  From 2^25 pixels the size includes the residual plane
 * (~1 byte per pixel) through which the equalize LUT_CORRECT entry points
 * (gpcx_lut_correct_device, gpcx_lut_correct_peer_device) move the image
 * from their count pass to their apply pass at 1 instead of 2 B/px; a
 * workspace of at least gpcx_lut_workspace_size(1, .) bytes (the fixed
 * part) is accepted by every call and only gives up that plane. */
int gpcx_lut_workspace_size(uint64_t n, uint64_t* bytes);
/* 65536-bin u32 histogram of n u16 samples (n < 2^32). */
int gpcx_lut_hist_device(const uint16_t* img, uint64_t n, uint32_t* hist,
                         void* ws, uint64_t ws_bytes, void* stream);
/* LUT (65536 x u16) + stats from a histogram (stats: device pointer); ws is
 * a LUT workspace (scratch for the per-slice scan summaries). */
int gpcx_lut_from_hist_device(const uint32_t* hist, int mode, uint16_t* lut,
                              gpcx_lut_stats* stats, void* ws, uint64_t ws_bytes,
                              void* stream);
/* The second half of a row-band sharded LUT_CORRECT: LUT + stats from the
 * merged (all-reduced) histogram, then out = LUT[in] over this band -- one
 * kernel launch when in/out are 16-byte co-aligned (in == out allowed). */
int gpcx_lut_correct_from_hist_device(const uint32_t* hist, int mode,
                                      const uint16_t* in, uint16_t* out,
                                      uint64_t n, uint16_t* lut,
                                      gpcx_lut_stats* stats, void* ws,
                                      uint64_t ws_bytes, void* stream);
/* min/max statistics only (stretch mode's reduction); stats device ptr. */
int gpcx_lut_minmax_device(const uint16_t* img, uint64_t n,
                           gpcx_lut_stats* stats, void* ws, uint64_t ws_bytes,
                           void* stream);
/* LUT from stats (stretch mode). */
int gpcx_lut_from_minmax_device(const gpcx_lut_stats* stats, uint16_t* lut,
                                void* stream);
int gpcx_lut_gen_device(const uint16_t* img, uint64_t n, int mode,
                        uint16_t* lut, gpcx_lut_stats* stats, void* ws,
                        uint64_t ws_bytes, void* stream);
/* out[i] = lut[in[i]] (in == out allowed). */
int gpcx_lut_apply_device(const uint16_t* lut, const uint16_t* in,
                          uint16_t* out, uint64_t n, void* stream);
/* LUT_GEN then LUT_APPLY on the same image. */
int gpcx_lut_correct_device(const uint16_t* in, uint16_t* out, uint64_t n,
                            int mode, uint16_t* lut, gpcx_lut_stats* stats,
                            void* ws, uint64_t ws_bytes, void* stream);

/* Row-band sharded LUT_CORRECT / LUT_GEN with one process per GPU and the
 * histogram exchange fused into the kernel over peer memory (no NCCL; the
 * reference has no multi-GPU path -- SURVEY.md §8e's "one exchange step").
 *   1. every rank: gpcx_lut_peer_create(rank, nranks, &p) on its device and
 *      gpcx_lut_peer_ipc_handle(p, h) (GPCX_IPC_HANDLE_BYTES bytes);
 *   2. the handles are all-gathered by the caller (torch.distributed, MPI,
 *      a file ...) in rank order and passed to gpcx_lut_peer_connect;
 *   3. every rank issues the SAME sequence of gpcx_lut_correct_peer_device
 *      calls on its band (out == NULL: LUT + stats only).  Each call is one
 *      cooperative launch: count the band, publish it, meet the peers
 *      (system-scope flags), sum their histograms with P2P loads, build the
 *      identical LUT on every rank, apply it to the band.
 * A rank whose peers never arrive traps after GPCX_PEER_TIMEOUT_MS (default
 * 60000) and the call's stream reports the failure.
 * Sizes: each rank's band n < 2^32 (its own histogram is u32); the group's
 * summed histogram, its totals, cdf_min and stats.n are 64-bit, so the whole
 * image may hold up to nranks * (2^32 - 1) pixels (8 ranks: ~2^35, e.g. a
 * 131072 x 262143 scene).  (gpcx_lut_correct_from_hist_device takes a u32
 * histogram: a caller that all-reduces band histograms itself must keep the
 * image below 2^32 pixels or pass per-bin sums that fit in u32.) */
#define GPCX_IPC_HANDLE_BYTES 64
typedef struct gpcx_lut_peer gpcx_lut_peer;
int gpcx_lut_peer_create(int rank, int nranks, gpcx_lut_peer** out);
int gpcx_lut_peer_ipc_handle(const gpcx_lut_peer* p, void* handle);
int gpcx_lut_peer_connect(gpcx_lut_peer* p, const void* handles);
int gpcx_lut_peer_destroy(gpcx_lut_peer* p);
int gpcx_lut_correct_peer_device(gpcx_lut_peer* p, const uint16_t* in, uint16_t* out,
                                 uint64_t n, int mode, uint16_t* lut,
                                 gpcx_lut_stats* stats, void* ws, uint64_t ws_bytes,
                                 void* stream);

/* C (m x n) = A (m x k) * B (k x n), all f32 row-major with leading
 * dimensions lda/ldb/ldc (elements).  prec selects the path (GPCX_PREC_*).
 * Workspace: required for TF32 / BF16 (prepared operands); optional for
 * F32, where it holds A^T for the fastest SIMT kernel (same bits without). */
int gpcx_matmul_workspace_size(int prec, uint64_t m, uint64_t n, uint64_t k,
                               uint64_t* bytes);
int gpcx_matmul_device(int prec, uint64_t m, uint64_t n, uint64_t k,
                       const float* A, uint64_t lda, const float* B,
                       uint64_t ldb, float* C, uint64_t ldc, void* ws,
                       uint64_t ws_bytes, void* stream);

/* Synthetic inputs, bit-identical to oracle/: rows
 * [row0, row0 + nrows) of a rows x cols image / matrix. */
int gpcx_synth_image_device(int kind, uint64_t seed, uint64_t rows,
                            uint64_t cols, uint64_t row0, uint64_t nrows,
                            uint16_t* out, void* stream);
int gpcx_synth_matrix_device(int kind, uint64_t seed, uint64_t rows,
                             uint64_t cols, uint64_t row0, uint64_t nrows,
                             float* out, void* stream);
/* BAYER_BILINEAR (gradient = 0) / BAYER_GRADIENT (gradient = 1) on a device
 * rows x cols u16 mosaic -> out = R || G || B planes (3 * rows * cols u16);
 * phase = 0 RGGB, 1 BGGR, 2 GRBG, 3 GBRG (gpc::img::CfaPhase order). */
int gpcx_demosaic_device(int gradient, int phase, const uint16_t* in, uint16_t* out,
                         uint64_t rows, uint64_t cols, void* stream);

/* DEVINFO: the reference's 12-attribute record (proj/include/gpc/devinfo.hpp:23-38). */
typedef struct gpcx_device_info {
  char name[256];
  char compute_capability[16];
  int32_t warp_size;
  uint64_t total_constant_memory;
  uint64_t total_global_memory;
  uint64_t shared_memory_per_block;
  int64_t clock_rate_khz;
  int32_t multi_processor_count;
  int32_t registers_per_block;
  int32_t max_threads_per_block;
  int32_t max_grid_size[3];
  int32_t max_threads_dim[3];
} gpcx_device_info;
/* Records of the bound devices (cap entries max; *count = number found). */
int gpcx_devinfo_probe(gpcx_device_info* out, int cap, int* count);
/* The reference's canonical XML for n records (proj/src/devinfo.cpp:94-125);
 * *len = bytes needed (excluding the NUL); fails SIZE_MISMATCH if cap is too small. */
int gpcx_devinfo_render(const gpcx_device_info* devs, int n, char* out, uint64_t cap,
                        uint64_t* len);

/* digest += sum_i splitmix64(((index0 + i) << 16) | v[i])  (device u64). */
int gpcx_digest_u16_device(const uint16_t* v, uint64_t n, uint64_t index0,
                           uint64_t* digest, void* stream);

/* ------------------------------------------------------------------ */
/* Executor: the B200 task server (replaces srv::Server,               */
/* proj/include/gpc/server.hpp:49-84).  Same wire contract; inside, a   */
/* staged pipeline: epoll front end (header, one parse, admission       */
/* control) -> payload receive into pinned staging -> one queue and     */
/* worker group per bound GPU -> response send (csrc/host/server.hpp).  */
/* ------------------------------------------------------------------ */

/* Start a server on bind_addr:port (port 0 = ephemeral; *bound_port gets
 * the real one).  max_tasks <= 0 means 2 x hardware threads as in the
 * reference (server.cpp:114-119): the number of handlers running at once
 * (split over the bound devices).  idle_timeout_ms <= 0 means 30000.  At
 * most GPCX_MAX_PENDING (default max(64, 4 x max_tasks)) admitted requests
 * are in progress; the next is answered ERR:TASK_FAILED, msg "server busy
 * ..." before its payload is read. */
int gpcx_server_start(const char* bind_addr, uint16_t port, int max_tasks,
                      int idle_timeout_ms, void** handle,
                      uint16_t* bound_port);
int gpcx_server_stop(void* handle);
/* Cumulative phase times of the requests a running server answered:
 * payload received | remaining task work after the last payload byte |
 * response written (milliseconds, summed over requests). */
typedef struct gpcx_server_stats {
  uint64_t requests;
  double recv_ms, task_ms, send_ms;
  uint64_t busy;     /* answered ERR:TASK_FAILED "server busy" by admission control */
  uint64_t dropped;  /* connections closed without a response (idle, cut short, I/O) */
} gpcx_server_stats;
int gpcx_server_stats_get(void* handle, gpcx_server_stats* out);
/* Serve one request held in memory with the server's admission and error
 * rules (the reference's handle_connection over a buffer, server.cpp:51-112).  Writes the response frame bytes
 * to resp (resp_cap must hold it; *resp_len = bytes needed).  Returns the
 * transport status (TRUNCATED for a cut-off request), 0 when answered. */
int gpcx_handle_request(const uint8_t* req, uint64_t req_len, uint8_t* resp,
                        uint64_t resp_cap, uint64_t* resp_len);

/* Client side (the reference's client::submit, proj/src/client.cpp:97-129):
 * one request over one TCP connection.  The payload is the concatenation of
 * nparts buffers (parts[i], part_len[i]) -- e.g. LUT || image without a
 * copy.  The response payload lands in resp (resp_cap bytes; *resp_len =
 * its size, SIZE_MISMATCH if it does not fit); status and params are
 * written NUL-terminated into the given buffers (64 and 256 bytes
 * suffice).  An ERR:<CODE> response is data (returns OK);
 * transport failures return CONNECT_FAILED / TRUNCATED / IO_ERROR. */
int gpcx_client_submit(const char* host, uint16_t port, const char* flag, const char* params,
                       const void* const* parts, const uint64_t* part_len, int nparts,
                       const char* output_name, void* resp, uint64_t resp_cap,
                       uint64_t* resp_len, char* status, uint64_t status_cap,
                       char* resp_params, uint64_t resp_params_cap);

#ifdef __cplusplus
}
#endif

#endif /* GPCX_H */
