// Grid-barrier latency on B200 with 132 persistent CTAs (clusters of 4):
//  A: every CTA release-adds one counter, thread 0 acquire-polls it
//  B: cluster barrier, then rank 0 of each cluster adds/polls, cluster barrier again
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_flat(unsigned int* ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned int v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory"); } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

template <int MODE>
__global__ void k(unsigned int* ctr, int reps, long long* out, double* junk) {
  cg::cluster_group cl = cg::this_cluster();
  const int nclu = gridDim.x / cl.num_blocks();
  long long t0 = clock64();
  for (int i = 1; i <= reps; ++i) {
    if (MODE == 2) junk[(blockIdx.x * 256 + threadIdx.x) * 2] = i;   // pending stores to drain
    if (MODE == 0 || MODE == 2) {
      bar_flat(ctr, (unsigned)i * gridDim.x);
    } else {
      cl.sync();
      if (cl.block_rank() == 0) bar_flat(ctr, (unsigned)i * nclu);   // note: __syncthreads inside only this CTA
      cl.sync();
    }
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[MODE] = (t1 - t0) / reps;
}

int main() {
  unsigned int* ctr; long long* out; double* junk;
  cudaMalloc(&ctr, 4096); cudaMalloc(&out, 64); cudaMalloc(&junk, 1 << 24);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(ctr, 0, 4096);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
    cfg.gridDim = dim3(132); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 0; cfg.attrs = at; cfg.numAttrs = 2;
    cudaError_t e;
    if (mode == 0) e = cudaLaunchKernelEx(&cfg, k<0>, ctr, 200, out, junk);
    else if (mode == 1) e = cudaLaunchKernelEx(&cfg, k<1>, ctr, 200, out, junk);
    else e = cudaLaunchKernelEx(&cfg, k<2>, ctr, 200, out, junk);
    cudaError_t e2 = cudaDeviceSynchronize();
    long long h[3];
    cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %lld cycles per barrier (%s / %s)\n", mode,
           mode == 0 ? "flat, 132 arrivals" : mode == 1 ? "cluster-hierarchical, 33 arrivals" : "flat with a pending store per thread",
           h[mode], cudaGetErrorString(e), cudaGetErrorString(e2));
  }
  return 0;
}
