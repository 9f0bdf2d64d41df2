// bw_probe.cu -- HBM ceilings for the write-heavy image kernels (design
// exploration for demosaic.cu; not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe tools/bw_probe.cu
// Each kernel moves the demosaic's bytes at 16384^2 (2 B in, 6 B out per px)
// without the stencil, so the gap to demosaic_kernel is the stencil's cost.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// write-only, grid-stride
__global__ void wr(uint4* out, uint64_t nvec) {
  const uint4 z = make_uint4(threadIdx.x, 1, 2, 3);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) __stcs(out + i, z);
}
// 1 in : 3 out (planes), grid-stride, CS stores
template <bool CS>
__global__ void r1w3(const uint4* in, uint4* out, uint64_t nvec) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 q = ldnc(in + i);
    if (CS) { __stcs(out + i, q); __stcs(out + nvec + i, q); __stcs(out + 2 * nvec + i, q); }
    else { out[i] = q; out[nvec + i] = q; out[2 * nvec + i] = q; }
  }
}
// 1 in : 3 out, one-shot CTAs laid out like demosaic (16 rows x 256 cols tile, 256 threads, 2 rows each)
__global__ void r1w3_tile(const uint16_t* in, uint16_t* out, int cols, uint64_t plane) {
  const int r0 = blockIdx.y * 16 + 2 * (threadIdx.x >> 5), c = blockIdx.x * 256 + 8 * (threadIdx.x & 31);
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const uint64_t off = (uint64_t)(r0 + rr) * cols + c;
    const uint4 q = ldnc((const uint4*)(in + off));
    __stcs((uint4*)(out + off), q);
    __stcs((uint4*)(out + plane + off), q);
    __stcs((uint4*)(out + 2 * plane + off), q);
  }
}
// 1:1 copy
__global__ void cp(const uint4* in, uint4* out, uint64_t nvec) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) __stcs(out + i, ldnc(in + i));
}

template <class F>
float time(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 8; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (r > 0 && ms < best) best = ms;
  }
  return best;
}

int main() {
  const int rows = 16384, cols = 16384;
  const uint64_t n = (uint64_t)rows * cols, nvec = n / 8;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint16_t *in, *out;
  CK(cudaMalloc(&in, n * 2)); CK(cudaMalloc(&out, n * 6));
  CK(cudaMemset(in, 1, n * 2)); CK(cudaMemset(out, 0, n * 6));
  auto rep = [&](const char* name, float ms, double bytes) { printf("%-40s %8.4f ms %8.1f GB/s\n", name, ms, bytes / ms / 1e6); };
  for (int k : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "write-only 6B/px  grid %dx148x256", k);
    rep(nm, time([&] { wr<<<k * sms, 256>>>((uint4*)out, 3 * nvec); }), 6.0 * n);
    snprintf(nm, 64, "r1w3 cs  grid %dx148x256", k);
    rep(nm, time([&] { r1w3<true><<<k * sms, 256>>>((const uint4*)in, (uint4*)out, nvec); }), 8.0 * n);
    snprintf(nm, 64, "r1w3 wb  grid %dx148x256", k);
    rep(nm, time([&] { r1w3<false><<<k * sms, 256>>>((const uint4*)in, (uint4*)out, nvec); }), 8.0 * n);
    snprintf(nm, 64, "copy 4B/px grid %dx148x256", k);
    rep(nm, time([&] { cp<<<k * sms, 256>>>((const uint4*)in, (uint4*)out, nvec); }), 4.0 * n);
  }
  rep("memset 6B/px", time([&] { cudaMemsetAsync(out, 3, n * 6); }), 6.0 * n);
  rep("r1w3 one-shot 16x256 tiles", time([&] { r1w3_tile<<<dim3(cols / 256, rows / 16), 256>>>(in, out, cols, n); }), 8.0 * n);
  return 0;
}
