// fused_trace.cu -- per-phase timeline of lut.cu's fused_kernel (globaltimer
// stamps of thread 0 of every CTA; design exploration, not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DGPCX_LUT_TRACE \
//        -o tools/fused_trace tools/fused_trace.cu paper_1505_05655_b200/csrc/status.cpp
//   ./tools/fused_trace [rows cols [r|u]]   (bench.py's ramp12 / uniform16 scenes, c: constant)   (GPCX_LUT_PLANE=0: no residual plane)
#include "../paper_1505_05655_b200/csrc/lut.cu"
#include "../paper_1505_05655_b200/csrc/synth.cu"  // the bench's ramp12 / uniform16 scenes

// the library's device-health hook (host/runtime.cpp) is not linked here
namespace gpcx::rt {
void note_cuda_error(cudaError_t, const char*) {}
}  // namespace gpcx::rt

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void fill_kernel(std::uint16_t* p, std::uint64_t n, std::uint16_t v) {
  for (std::uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += 1024ull * 256) p[i] = v;
}

int main(int argc, char** argv) {
  const std::uint64_t rows = argc > 2 ? std::strtoull(argv[1], nullptr, 10) : 4096;
  const std::uint64_t cols = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 4096;
  const char kc = argc > 3 ? argv[3][0] : 'r';
  const int kind = kc == 'u' ? 1 : 0;  // r: ramp12, u: uniform16 (seed 0x5eed), c: constant 1234
  const std::uint64_t n = rows * cols;
  std::uint16_t *img, *out, *lut;
  void* ws;
  gpcx_lut_stats* stats;
  unsigned long long* trace;
  cudaMalloc(&img, n * 2);
  cudaMalloc(&out, n * 2);
  cudaMalloc(&lut, 131072);
  cudaMalloc(&stats, sizeof(gpcx_lut_stats));
  const std::uint64_t ws_bytes = gpcx::lut::workspace_bytes(n);  // room for the residual plane
  cudaMalloc(&ws, ws_bytes);
  cudaMemset(ws, 0, ws_bytes);
  const int sms = gpcx::device_sm_count();
  cudaMalloc(&trace, sms * 16 * 8);
  cudaMemcpyToSymbol(gpcx::lut::g_lut_trace, &trace, sizeof(trace));
  gpcx::synth::launch_image(kind, 0x5EED, rows, cols, 0, rows, img, nullptr);
  if (kc == 'c') fill_kernel<<<1024, 256>>>(img, n, 1234);
  cudaDeviceSynchronize();
  char* flush;
  cudaMalloc(&flush, 512 << 20);
  const char* names[] = {"start", "counted", "flushed", "sync1", "merged", "sync2",
                         "lut", "sync3", "lut->smem", "applied"};
  std::vector<unsigned long long> t(sms * 16);
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemset(trace, 0, sms * 16 * 8);
    cudaMemset(flush, rep, 512 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    gpcx::lut::launch_correct(img, out, n, GPCX_LUT_EQUALIZE, lut, stats, ws, nullptr, ws_bytes);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(t.data(), trace, t.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < sms; ++c) t0 = std::min(t0, t[c * 16]);
    std::printf("rep %d: events %.2f us (%s)\n", rep, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    for (int k = 0; k < 10; ++k) {
      double mn = 1e30, mx = 0, sum = 0;
      int cnt = 0;
      for (int c = 0; c < sms; ++c) {
        if (t[c * 16 + k] == 0) continue;
        const double v = (t[c * 16 + k] - t0) * 1e-3;
        mn = std::min(mn, v);
        mx = std::max(mx, v);
        sum += v;
        ++cnt;
      }
      if (cnt) std::printf("  %-10s min %7.2f  avg %7.2f  max %7.2f us  (%d CTAs)\n", names[k], mn,
                           sum / cnt, mx, cnt);
    }
    if (rep == 3 && std::getenv("TRACE_CTAS") != nullptr) {  // per-CTA end of the count pass
      std::printf("  counted per CTA (us):");
      for (int c = 0; c < sms; ++c) std::printf(" %d:%.1f", c, (t[c * 16 + 1] - t0) * 1e-3);
      std::printf("\n");
    }
  }
  return 0;
}
