// How many clusters of 2/4/8 CTAs (1 CTA per SM: ~211 KB dynamic smem) can be co-resident?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe/clusters tools/probe/clusters.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) { if (threadIdx.x == 0) out[blockIdx.x] = 1; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 216 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms / cs * cs);
    cfg.blockDim = dim3(224);
    cfg.dynamicSmemBytes = 216 * 1024;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cs;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d -> %d CTAs of %d SMs (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
  }
}
