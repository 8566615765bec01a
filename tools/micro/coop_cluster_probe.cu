// Probe: cooperative launch combined with thread-block clusters on sm_100a
// (cudaLaunchKernelEx with cluster dimension + cooperative attribute), one CTA
// per SM via large dynamic shared memory; a DSMEM read inside the cluster and a
// grid-wide monotonic barrier.  Prints max active clusters and the result.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(8, 1, 1) k_probe(unsigned* bar, int* out) {
  extern __shared__ int sm[];
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  cl.sync();
  int* peer = cl.map_shared_rank(sm, (cl.block_rank() + 1) % cl.num_blocks());
  int v = peer[0];
  cl.sync();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (atomicAdd(bar, 0u) < gridDim.x) __nanosleep(64);
    out[blockIdx.x] = v;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 180 * 1024;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 8; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cfg.gridDim = dim3(8);
  int nclusters = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, k_probe, &cfg);
  printf("SMs %d, max active clusters of 8 (1 CTA/SM): %d (%s)\n", sms, nclusters, cudaGetErrorString(e));
  for (int ncl : {nclusters, nclusters + 1}) {
    unsigned* bar; int* out;
    cudaMalloc(&bar, 4); cudaMemset(bar, 0, 4);
    cudaMalloc(&out, 4 * 8 * ncl);
    cudaLaunchAttribute at2[2];
    at2[0] = attr[0];
    at2[1].id = cudaLaunchAttributeCooperative; at2[1].val.cooperative = 1;
    cfg.attrs = at2; cfg.numAttrs = 2;
    cfg.gridDim = dim3(8 * ncl);
    e = cudaLaunchKernelEx(&cfg, k_probe, bar, out);
    cudaError_t e2 = cudaDeviceSynchronize();
    int h[8] = {0};
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("grid %d CTAs: launch %s, sync %s, out[0..7] = %d %d %d %d %d %d %d %d\n", 8 * ncl, cudaGetErrorString(e),
           cudaGetErrorString(e2), h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    cudaGetLastError();
  }
  return 0;
}
