// Probe: how many clusters of a pass-kernel-shaped CTA can be co-resident (cluster placement limit).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}
int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem_kb : {100, 150, 197, 215})
    for (int cl : {1, 2, 3, 4, 6, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cl * 64);
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = smem_kb * 1024;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = cl;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
      printf("smem %d KB cluster %d: max active clusters %d (%d SMs) %s\n", smem_kb, cl, n, n * cl,
             e ? cudaGetErrorString(e) : "");
    }
}
