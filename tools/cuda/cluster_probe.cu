// cluster_probe.cu -- how many thread-block clusters of 2..16 CTAs of the tree kernels' shape (512
// threads, 64 registers, 2 resident blocks per SM) fit co-resident on this GPU
// (cudaOccupancyMaxActiveClusters), against the 2 x SM-count blocks of today's cooperative grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cp tools/cuda/cluster_probe.cu && /tmp/cp
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 2) k_shape(unsigned* out) {
  unsigned v[40];
#pragma unroll
  for (int i = 0; i < 40; i++) v[i] = out[threadIdx.x * 40 + i] * (i + 3);   // keep registers live
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 40; i++) s += v[i] * v[(i + 7) % 40];
  out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_shape, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_shape);
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_shape, 512, 0);
  printf("SMs %d, registers %d, blocks/SM %d -> cooperative grid %d blocks\n", sms, fa.numRegs, bps, bps * sms);
  for (int c = 2; c <= 16; c *= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * 64);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_shape, &cfg);
    printf("cluster %2d: max active clusters %4d -> %4d blocks (%s)\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
