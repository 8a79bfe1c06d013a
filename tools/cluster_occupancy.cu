// Probe: how many clusters of 1/2/4/8 CTAs (one CTA per SM, ~200 KB of shared
// memory each) can be co-resident on this device (cudaOccupancyMaxActiveClusters).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; if (threadIdx.x == 1000) s[0] = 0; }
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int c : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(sms / c * c));
    cfg.blockDim = dim3(640);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = c;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: %3d clusters resident = %3d CTAs of %d SMs (%s)\n", c, n, n * c, sms,
           cudaGetErrorString(e));
  }
  return 0;
}
