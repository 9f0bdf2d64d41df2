// apply_bench.cu -- LUT-apply kernel variants on sm_100a (design exploration
// for lut.cu's apply_kernel; not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/apply_bench tools/apply_bench.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void gen(uint16_t* out, uint64_t n, int kind) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = sm64(0x5eed ^ i);
    out[i] = kind ? (h & 0xFFFF) : (1024 + ((i >> 15) + (i & 32767)) / 21 + (h >> 58));
  }
}
__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stna(uint4* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void stcs(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 look(const uint16_t* s, uint4 q) {
  uint4 r;
  r.x = s[q.x & 0xFFFF] | ((uint32_t)s[q.x >> 16] << 16);
  r.y = s[q.y & 0xFFFF] | ((uint32_t)s[q.y >> 16] << 16);
  r.z = s[q.z & 0xFFFF] | ((uint32_t)s[q.z >> 16] << 16);
  r.w = s[q.w & 0xFFFF] | ((uint32_t)s[q.w >> 16] << 16);
  return r;
}

// MODE 0: plain grid-stride unroll U (current product)
// MODE 1: software pipelined: loads of group g+1 in flight while group g is looked up
// MODE 2: like 0 with st.global.cs
// MODE 3: contiguous chunk per CTA (block-cyclic 4 KiB tiles) instead of grid-stride
template <int MODE, int THREADS, int U>
__global__ void __launch_bounds__(THREADS, 1) apply(const uint16_t* lut, const uint16_t* in, uint16_t* out, uint64_t n) {
  extern __shared__ uint4 sm[];
  for (int i = threadIdx.x; i < 8192; i += THREADS) sm[i] = ((const uint4*)lut)[i];
  __syncthreads();
  const uint16_t* s = (const uint16_t*)sm;
  const uint4* src = (const uint4*)in;
  uint4* dst = (uint4*)out;
  const uint64_t nvec = n / 8, stride = (uint64_t)gridDim.x * THREADS;
  uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
  if (MODE == 0 || MODE == 2) {
    for (; i + (U - 1) * stride < nvec; i += U * stride) {
      uint4 q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) q[u] = ldnc(src + i + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (MODE == 2) stcs(dst + i + u * stride, look(s, q[u]));
        else stna(dst + i + u * stride, look(s, q[u]));
      }
    }
    for (; i < nvec; i += stride) stna(dst + i, look(s, ldnc(src + i)));
  } else if (MODE == 1) {
    uint4 q[U], nq[U];
    bool have = i + (U - 1) * stride < nvec;
    if (have) {
#pragma unroll
      for (int u = 0; u < U; ++u) q[u] = ldnc(src + i + u * stride);
    }
    while (have) {
      const uint64_t nx = i + U * stride;
      const bool nhave = nx + (U - 1) * stride < nvec;
      if (nhave) {
#pragma unroll
        for (int u = 0; u < U; ++u) nq[u] = ldnc(src + nx + u * stride);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) stna(dst + i + u * stride, look(s, q[u]));
#pragma unroll
      for (int u = 0; u < U; ++u) q[u] = nq[u];
      i = nx;
      have = nhave;
    }
    for (; i < nvec; i += stride) stna(dst + i, look(s, ldnc(src + i)));
  } else {
    // each CTA walks whole 16 KiB tiles: tile t = blockIdx + k*grid
    const uint64_t tile_vec = THREADS * U;
    const uint64_t ntiles = nvec / tile_vec;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const uint64_t base = t * tile_vec + threadIdx.x;
      uint4 q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) q[u] = ldnc(src + base + u * THREADS);
#pragma unroll
      for (int u = 0; u < U; ++u) stna(dst + base + u * THREADS, look(s, q[u]));
    }
  }
}

template <int MODE, int THREADS, int U>
void run(const char* name, const uint16_t* lut, const uint16_t* in, uint16_t* out, uint64_t n, int grid) {
  cudaFuncSetAttribute(apply<MODE, THREADS, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    apply<MODE, THREADS, U><<<grid, THREADS, 131072>>>(lut, in, out, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
  }
  cudaError_t e = cudaGetLastError();
  printf("%-34s %8.4f ms  %7.1f GB/s %s\n", name, best, 4.0 * n / best / 1e6, e ? cudaGetErrorString(e) : "");
}

int main() {
  const uint64_t n = 32768ull * 32768ull;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint16_t *img, *out, *lut;
  CK(cudaMalloc(&img, n * 2)); CK(cudaMalloc(&out, n * 2)); CK(cudaMalloc(&lut, 131072));
  gen<<<4096, 256>>>(lut, 65536, 1);
  for (int kind = 0; kind < 2; ++kind) {
    gen<<<4096, 256>>>(img, n, kind);
    CK(cudaDeviceSynchronize());
    printf("== %s\n", kind ? "uniform16" : "ramp12");
    run<0, 1024, 4>("stride u4 t1024 (product)", lut, img, out, n, sms);
    run<0, 1024, 2>("stride u2 t1024", lut, img, out, n, sms);
    run<0, 512, 8>("stride u8 t512", lut, img, out, n, sms);
    run<1, 1024, 2>("pipelined u2 t1024", lut, img, out, n, sms);
    run<1, 512, 4>("pipelined u4 t512", lut, img, out, n, sms);
    run<2, 1024, 4>("stride u4 t1024 st.cs", lut, img, out, n, sms);
    run<3, 1024, 4>("tiles u4 t1024", lut, img, out, n, sms);
    run<3, 512, 8>("tiles u8 t512", lut, img, out, n, sms);
    cudaMemcpy(out, img, n * 2, cudaMemcpyDeviceToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); cudaMemcpy(out, img, n * 2, cudaMemcpyDeviceToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-34s %8.4f ms  %7.1f GB/s\n", "cudaMemcpy D2D", ms, 4.0 * n / ms / 1e6);
  }
  return 0;
}
