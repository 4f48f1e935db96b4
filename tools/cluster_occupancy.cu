// How many clusters of 2 / 4 / 8 CTAs (one 256-thread CTA with ~210 KB of
// shared memory per SM, the GEMM engine's footprint) the B200 co-schedules:
// the SM budget an operand-multicast cluster shape would give up.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}
int main() {
  const int smem = 12 * 16384 + 4 * 2 * 4096 + 1536;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * (sms / cs));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a;
    a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = cs;
    a.val.clusterDim.y = 1;
    a.val.clusterDim.z = 1;
    cfg.attrs = &a;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
    printf("cluster %2d: %3d clusters = %3d SMs of %d (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
  }
  return 0;
}
