// pipe_probe.cu -- can consecutive LUT_CORRECT requests overlap on one B200?
// (design exploration, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_probe tools/pipe_probe.cu
// The count pass of LUT_CORRECT is bound by the shared-memory atomic unit
// (~0.47 ms per 2^30 samples at 148 SMs, HBM at ~70%), the apply pass by HBM
// (~0.66 ms).  Running image i+1's count on x SMs while image i's apply runs
// on the other 148-x SMs (two streams, 1 CTA of 1024 threads per SM, 128 KiB
// smem each) would use both units at once.  This probe times, per image:
//   count alone | apply alone | count + apply back to back | both passes of
//   a stream of images with the SMs split x : 148-x.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen(uint16_t* out, uint64_t n, uint64_t cols) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = sm64(0x5eed ^ i), r = i / cols, c = i % cols;
    long long v = 1024 + (3071ull * (r + c)) / (2 * cols - 2) + ((long long)(h >> 58) - 32);
    out[i] = v;
  }
}

__device__ __forceinline__ uint4 ld(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st(uint4* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// red.shared on packed u16 pairs: the product's count rate (~0.48 ms per
// 2^30 samples, tools/hist_probe mode 0) without its wrap bookkeeping
__device__ __forceinline__ void cnt(uint32_t* bins, uint32_t v, uint32_t*) {
  const uint32_t addr = (uint32_t)__cvta_generic_to_shared(bins + (v >> 1));
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(1u << ((v & 1) << 4)) : "memory");
}

// count pass: grid-stride over the image, per-CTA packed u16 histogram,
// flushed to parts at the end (the product's phase 1)
__global__ void __launch_bounds__(1024, 1) count_k(const uint16_t* img, uint64_t n, uint32_t* parts, uint32_t* ovf) {
  extern __shared__ uint4 sm[];
  uint32_t* bins = (uint32_t*)sm;
  for (int i = threadIdx.x; i < 8192; i += 1024) sm[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const uint4* body = (const uint4*)img;
  const uint64_t nvec = n / 8, stride = (uint64_t)gridDim.x * 1024;
  auto vec = [&](uint4 q) {
    cnt(bins, q.x & 0xFFFF, ovf); cnt(bins, q.x >> 16, ovf); cnt(bins, q.y & 0xFFFF, ovf); cnt(bins, q.y >> 16, ovf);
    cnt(bins, q.z & 0xFFFF, ovf); cnt(bins, q.z >> 16, ovf); cnt(bins, q.w & 0xFFFF, ovf); cnt(bins, q.w >> 16, ovf);
  };
  uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
  for (; i + stride < nvec; i += 2 * stride) {
    uint4 a = ld(body + i), b = ld(body + i + stride);
    vec(a);
    vec(b);
  }
  for (; i < nvec; i += stride) vec(ld(body + i));
  __syncthreads();
  uint4* dst = (uint4*)(parts + (uint64_t)blockIdx.x * 32768);
  for (int j = threadIdx.x; j < 8192; j += 1024) dst[j] = sm[j];
}

__global__ void __launch_bounds__(1024, 1) apply_k(const uint16_t* lut, const uint16_t* in, uint16_t* out, uint64_t n) {
  extern __shared__ uint4 sm[];
  for (int i = threadIdx.x; i < 8192; i += 1024) sm[i] = ((const uint4*)lut)[i];
  __syncthreads();
  const uint16_t* s = (const uint16_t*)sm;
  const uint4* src = (const uint4*)in;
  uint4* dst = (uint4*)out;
  const uint64_t nvec = n / 8, stride = (uint64_t)gridDim.x * 1024;
  auto look = [&](uint4 q) {
    uint4 r;
    r.x = s[q.x & 0xFFFF] | (s[q.x >> 16] << 16); r.y = s[q.y & 0xFFFF] | (s[q.y >> 16] << 16);
    r.z = s[q.z & 0xFFFF] | (s[q.z >> 16] << 16); r.w = s[q.w & 0xFFFF] | (s[q.w >> 16] << 16);
    return r;
  };
  uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
  for (; i + stride < nvec; i += 2 * stride) {
    uint4 a = ld(src + i), b = ld(src + i + stride);
    st(dst + i, look(a));
    st(dst + i + stride, look(b));
  }
  for (; i < nvec; i += stride) st(dst + i, look(ld(src + i)));
}

int main() {
  const uint64_t rows = 32768, cols = 32768, n = rows * cols;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint16_t *img[2], *out, *lut;
  uint32_t *parts, *ovf;
  CK(cudaMalloc(&img[0], n * 2));
  CK(cudaMalloc(&img[1], n * 2));
  CK(cudaMalloc(&out, n * 2));
  CK(cudaMalloc(&lut, 131072));
  CK(cudaMalloc(&parts, 300ull * 131072));
  CK(cudaMalloc(&ovf, 65536 * 4));
  CK(cudaMemset(ovf, 0, 65536 * 4));
  CK(cudaMemset(lut, 0x5a, 131072));
  gen<<<4096, 256>>>(img[0], n, cols);
  gen<<<4096, 256>>>(img[1], n, cols);
  cudaFuncSetAttribute(count_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(apply_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  CK(cudaDeviceSynchronize());
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int R = 10;
  auto timed = [&](auto body) -> float {
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, 0);
      body();
      cudaEventRecord(b, 0);
      if (cudaEventSynchronize(b) != cudaSuccess) printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    return best / R;
  };
  const float tc = timed([&] { for (int r = 0; r < R; ++r) count_k<<<sms, 1024, 131072>>>(img[r & 1], n, parts, ovf); });
  const float ta = timed([&] { for (int r = 0; r < R; ++r) apply_k<<<sms, 1024, 131072>>>(lut, img[r & 1], out, n); });
  const float tca = timed([&] {
    for (int r = 0; r < R; ++r) {
      count_k<<<sms, 1024, 131072>>>(img[r & 1], n, parts, ovf);
      apply_k<<<sms, 1024, 131072>>>(lut, img[r & 1], out, n);
    }
  });
  printf("count alone %.4f ms | apply alone %.4f ms | back to back %.4f ms per image (6 B/px: %.0f GB/s)\n", tc, ta,
         tca, 6.0 * n / tca / 1e6);
  for (int x : {64, 74, 84, 94, 104, 114, 124, 134}) {
    // per image: count(i+1) on x SMs || apply(i) on sms-x SMs; a barrier
    // per image pair (events) models the LUT dependency
    cudaEvent_t ec, ea;
    cudaEventCreateWithFlags(&ec, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ea, cudaEventDisableTiming);
    const float t = timed([&] {
      cudaEventRecord(a, 0);
      cudaStreamWaitEvent(s1, a, 0);
      cudaStreamWaitEvent(s2, a, 0);
      for (int r = 0; r < R; ++r) {
        count_k<<<x, 1024, 131072, s1>>>(img[(r + 1) & 1], n, parts, ovf);
        apply_k<<<sms - x, 1024, 131072, s2>>>(lut, img[r & 1], out, n);
        cudaEventRecord(ec, s1);
        cudaEventRecord(ea, s2);
        cudaStreamWaitEvent(s1, ea, 0);
        cudaStreamWaitEvent(s2, ec, 0);
      }
      cudaEventRecord(ec, s1);
      cudaEventRecord(ea, s2);
      cudaStreamWaitEvent(0, ec, 0);
      cudaStreamWaitEvent(0, ea, 0);
    });
    printf("split count %3d SMs | apply %3d SMs: %.4f ms per image (6 B/px: %.0f GB/s)\n", x, sms - x, t,
           6.0 * n / t / 1e6);
  }
  return 0;
}
