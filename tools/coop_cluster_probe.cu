// Probe: can a grid of several 16-CTA clusters be launched cooperatively
// (co-residency guaranteed) with ~200 KB dynamic shared memory per CTA?
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int* out) {
  cg::grid_group g = cg::this_grid();
  cg::cluster_group c = cg::this_cluster();
  extern __shared__ double sm[];
  sm[threadIdx.x] = threadIdx.x;
  c.sync();
  g.sync();
  if (threadIdx.x == 0) atomicAdd(out, 1);
}
int main() {
  int* d;
  cudaMalloc(&d, 4);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {16, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int ncl = 0;
    cudaError_t e0 = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    printf("cluster %d: max active clusters %d (%s)\n", cs, ncl, cudaGetErrorString(e0));
    for (int nc = 1; nc <= ncl + 1; nc++) {
      cfg.gridDim = dim3(cs * nc);
      cfg.numAttrs = 2;
      cudaMemset(d, 0, 4);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
      cudaError_t e2 = cudaDeviceSynchronize();
      int h = 0;
      cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
      printf("  coop launch %d clusters: launch %s sync %s done %d\n", nc, cudaGetErrorString(e),
             cudaGetErrorString(e2), h);
      cudaGetLastError();
    }
  }
  return 0;
}
