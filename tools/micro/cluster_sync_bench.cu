// Microbenchmark: cost of cluster.sync() and of a DSMEM all-gather step in 8- and 16-CTA
// clusters on B200 (sm_100a).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void sync_only(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = clock64() - t0;
}
__global__ void sync_gather(int iters, long long* out, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[2][64];
  const int n = cl.num_blocks();
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 64) buf[i & 1][threadIdx.x] = i + threadIdx.x;
    cl.sync();
    if (threadIdx.x < 64) {
      double v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = r < n ? cl.map_shared_rank(&buf[i & 1][0], r)[threadIdx.x] : 0.0;
#pragma unroll
      for (int r = 0; r < 16; ++r) acc += v[r];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = clock64() - t0;
  if (acc == -1.0) sink[0] = acc;
  cl.sync();
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 8);
  for (int csize : {2, 4, 8, 16}) {
    for (int threads : {256, 512}) {
      for (int which = 0; which < 2; ++which) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(csize);
        cfg.blockDim = dim3(threads);
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = csize;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        if (csize > 8) {
          cudaFuncSetAttribute(sync_only, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
          cudaFuncSetAttribute(sync_gather, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
        const int iters = 2000;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaError_t err;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (which == 0) err = cudaLaunchKernelEx(&cfg, sync_only, iters, d);
          else err = cudaLaunchKernelEx(&cfg, sync_gather, iters, d, s);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        long long cyc = 0;
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        printf("cluster %2d threads %3d %-12s: %6.3f us per iteration (%lld cycles) %s\n", csize, threads,
               which ? "sync+gather" : "sync", ms * 1e3 / iters, cyc / iters, cudaGetErrorString(err));
      }
    }
  }
  return 0;
}
