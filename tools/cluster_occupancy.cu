// How many clusters of size 2 / 4 / 8 / 16 fit at once with the limb GEMM's
// shared-memory footprint (cudaOccupancyMaxActiveClusters): a cluster size
// that leaves SMs idle cannot pay for TMA multicast of the A tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a tools/cluster_occupancy.cu -o /tmp/co && /tmp/co
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[0] = s[0];
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int smem_sizes[] = {1024, 100 * 1024, 197888};
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("{\"sms\": %d, \"results\": [", prop.multiProcessorCount);
  bool first = true;
  for (int smem : smem_sizes)
    for (int cs : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64);
      cfg.blockDim = dim3(320);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
      printf("%s{\"smem\": %d, \"cluster\": %d, \"max_active_clusters\": %d, \"sms_used\": %d, \"err\": \"%s\"}",
             first ? "" : ", ", smem, cs, n, n * cs, cudaGetErrorString(e));
      first = false;
    }
  printf("]}\n");
  return 0;
}
