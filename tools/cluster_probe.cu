// cluster_probe.cu -- how many SMs can a persistent kernel with 1 CTA per SM
// (200 KiB smem) occupy at cluster sizes 1 / 2 / 4 / 8 on this GPU?
// (cudaOccupancyMaxActiveClusters; design input for tc_gemm.cu's cluster choice)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/cluster_probe tools/cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* p) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  if (p) p[blockIdx.x] = s[threadIdx.x];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("SMs %d; persistent kernel, 1 CTA/SM (%d KiB smem)\n", sms, smem / 1024);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d SMs busy (%s)\n", cs, n, n * cs,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  }
  return 0;
}
