// hist_bench.cu -- microbenchmark of shared-memory histogram strategies on
// sm_100a (design exploration for lut.cu's hist_kernel; not product code).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hist_bench tools/hist_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen(uint16_t* out, uint64_t n, int kind, uint64_t cols) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = sm64(0x5eed ^ i);
    if (kind) out[i] = h & 0xFFFF;
    else { uint64_t r = i / cols, c = i % cols; long long v = 1024 + (3071ull * (r + c)) / (2 * cols - 2) + ((long long)(h >> 58) - 32); out[i] = v; }
  }
}

__device__ __forceinline__ uint4 ldnc(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// MODE 0: atom with return + overflow check (current product)
// MODE 1: atom, return unused (RED)
// MODE 2: loads only (xor sink)
// MODE 3: red via inline PTX red.shared.add.u32
// MODE 4: pair-merge: if both halves of a u32 land in the same word, one atom
template <int MODE, int THREADS, bool PIPE = false>
__global__ void __launch_bounds__(THREADS, 1) hist(const uint16_t* img, uint64_t n, uint32_t* parts, uint32_t* ovf) {
  extern __shared__ uint4 sm[];
  uint32_t* bins = (uint32_t*)sm;
  for (int i = threadIdx.x; i < 8192; i += THREADS) sm[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const uint4* body = (const uint4*)img;
  uint64_t nvec = n / 8, stride = (uint64_t)gridDim.x * THREADS;
  uint32_t sink = 0;
  auto one = [&](uint32_t v) {
    if (MODE == 0) {
      uint32_t hb = v & 1, inc = hb ? 0x10000u : 1u, mask = hb ? 0xFFFF0000u : 0xFFFFu;
      uint32_t old = atomicAdd(&bins[v >> 1], inc);
      if ((old & mask) == mask) atomicAdd(&ovf[v], 65536u);
    } else if (MODE == 1) {
      atomicAdd(&bins[v >> 1], (v & 1) ? 0x10000u : 1u);
    } else if (MODE == 2) {
      sink ^= v;
    } else if (MODE == 3) {
      uint32_t addr = (uint32_t)__cvta_generic_to_shared(&bins[v >> 1]);
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(addr), "r"(1u << ((v & 1) << 4)));
    }
  };
  auto word = [&](uint32_t q) {
    if (MODE == 4) {
      uint32_t a = q & 0xFFFF, b = q >> 16;
      if ((a >> 1) == (b >> 1)) {
        atomicAdd(&bins[a >> 1], (1u << ((a & 1) << 4)) + (1u << ((b & 1) << 4)));
      } else {
        atomicAdd(&bins[a >> 1], 1u << ((a & 1) << 4));
        atomicAdd(&bins[b >> 1], 1u << ((b & 1) << 4));
      }
    } else {
      one(q & 0xFFFF);
      one(q >> 16);
    }
  };
  uint64_t i = blockIdx.x * (uint64_t)THREADS + threadIdx.x;
  if (PIPE) {  // loads of stage g+1 in flight while stage g is counted
    uint4 q[2], nq[2];
    bool have = i + stride < nvec;
    if (have) { q[0] = ldnc(body + i); q[1] = ldnc(body + i + stride); }
    while (have) {
      const uint64_t nx = i + 2 * stride;
      const bool nhave = nx + stride < nvec;
      if (nhave) { nq[0] = ldnc(body + nx); nq[1] = ldnc(body + nx + stride); }
#pragma unroll
      for (int u = 0; u < 2; ++u) { word(q[u].x); word(q[u].y); word(q[u].z); word(q[u].w); }
      q[0] = nq[0]; q[1] = nq[1];
      i = nx; have = nhave;
    }
  }
  for (; i + 3 * stride < nvec; i += 4 * stride) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = ldnc(body + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) { word(q[u].x); word(q[u].y); word(q[u].z); word(q[u].w); }
  }
  for (; i < nvec; i += stride) { uint4 q = ldnc(body + i); word(q.x); word(q.y); word(q.z); word(q.w); }
  if (sink == 0x12345678) ovf[0] = sink;
  __syncthreads();
  uint4* dst = (uint4*)(parts + (uint64_t)blockIdx.x * 32768);
  for (int j = threadIdx.x; j < 8192; j += THREADS) dst[j] = sm[j];
}

template <int MODE, int THREADS, bool PIPE = false>
int run(const char* name, const uint16_t* img, uint64_t n, uint32_t* parts, uint32_t* ovf, int sms) {
  CK(cudaFuncSetAttribute(hist<MODE, THREADS, PIPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> ts;
  for (int r = 0; r < 8; ++r) {
    cudaEventRecord(a);
    hist<MODE, THREADS, PIPE><<<sms, THREADS, 131072>>>(img, n, parts, ovf);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); ts.push_back(ms);
  }
  float best = 1e9; for (float t : ts) best = t < best ? t : best;
  printf("%-28s %8.4f ms  %7.1f GB/s\n", name, best, 2.0 * n / best / 1e6);
  return 0;
}

int main() {
  const uint64_t rows = 32768, cols = 32768, n = rows * cols;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint16_t* img; uint32_t *parts, *ovf;
  CK(cudaMalloc(&img, n * 2)); CK(cudaMalloc(&parts, 300ull * 131072)); CK(cudaMalloc(&ovf, 262144));
  for (int kind = 0; kind < 2; ++kind) {
    gen<<<4096, 256>>>(img, n, kind, cols);
    CK(cudaDeviceSynchronize());
    printf("== %s\n", kind ? "uniform16" : "ramp12");
    run<0, 1024>("atom+check 1024", img, n, parts, ovf, sms);
    run<0, 768>("atom+check 768", img, n, parts, ovf, sms);
    run<0, 512>("atom+check 512", img, n, parts, ovf, sms);
    run<1, 1024>("atom noret 1024", img, n, parts, ovf, sms);
    run<2, 1024>("loads only 1024", img, n, parts, ovf, sms);
    run<3, 1024>("red.shared 1024", img, n, parts, ovf, sms);
    run<4, 1024>("pair-merge 1024", img, n, parts, ovf, sms);
    run<0, 1024, true>("atom+check 1024 pipelined", img, n, parts, ovf, sms);
    run<1, 1024, true>("atom noret 1024 pipelined", img, n, parts, ovf, sms);
    run<0, 768, true>("atom+check 768 pipelined", img, n, parts, ovf, sms);
  }
  return 0;
}
