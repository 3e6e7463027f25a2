// Design microbenchmarks for the ALS/hSVD kernels on B200 (sm_100a).
// Measures: fp64 FFMA peak, DMMA (mma.sync f64) peak, grid.sync latency,
// flag-barrier latency, L2-resident read bandwidth, DSMEM read bandwidth,
// CUDA-graph kernel-node latency.  Prints one line per measurement.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void ffma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

// m16n8k16 f64: A 8 regs, B 4 regs, C/D 4 regs
__global__ void dmma16_kernel(double* out, int iters) {
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%4,%4,%4,%4,%4,%4,%4}, {%5,%5,%5,%5}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void gridsync_kernel(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double x = 0;
  for (int i = 0; i < iters; ++i) { x += 1; g.sync(); }
  if (x == -1) sink[0] = x;
}

// sense-reversal flag barrier: one arrive per CTA, spin on generation
__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;
__global__ void flagbar_kernel(int iters, double* sink) {
  unsigned int nb = gridDim.x;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int gen = g_gen;
      __threadfence();
      unsigned int prev = atomicAdd(&g_count, 1u);
      if (prev == nb - 1) { g_count = 0; __threadfence(); g_gen = gen + 1; }
      else { while (g_gen == gen) { } }
      __threadfence();
    }
    __syncthreads();
  }
}

__global__ void l2read_kernel(const double2* __restrict__ buf, size_t n2, int iters, double* sink) {
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(buf + i);
      acc += v.x + v.y;
    }
  }
  if (acc == -1) sink[0] = acc;
}

// each CTA reads `words` doubles from the next CTA's shared memory in the cluster
__global__ void dsmem_kernel(int words, int iters, double* sink) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = i;
  cl.sync();
  unsigned int rank = cl.block_rank();
  double* remote = cl.map_shared_rank(sm, (rank + 1) % cl.num_blocks());
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = threadIdx.x * 2; i < words; i += blockDim.x * 2) {
      double2 v = *reinterpret_cast<double2*>(remote + i);
      acc += v.x + v.y;
    }
  }
  cl.sync();
  if (acc == -1) sink[0] = acc;
}

__global__ void clsync_kernel(int iters, double* sink) {
  cg::cluster_group cl = cg::this_cluster();
  double x = 0;
  for (int i = 0; i < iters; ++i) { x += 1; cl.sync(); }
  if (x == -1) sink[0] = x;
}

__global__ void empty_kernel(double* p) { if (threadIdx.x == 1000000) p[0] = 1; }

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("device %s sms=%d clock_khz=%d l2=%d smem_optin=%zu\n", prop.name, sms, prop.clockRate,
         prop.l2CacheSize, prop.sharedMemPerBlockOptin);
  double* d; CK(cudaMalloc(&d, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;

  // FFMA
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    ffma_kernel<<<blocks, threads>>>(d, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); ffma_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("ffma_f64_tflops %.2f (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  // DMMA m8n8k4
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    dmma_kernel<<<blocks, threads>>>(d, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("dmma_m8n8k4_tflops %.2f (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  {
    int iters = 2048, blocks = sms * 8, threads = 256;
    dmma16_kernel<<<blocks, threads>>>(d, 16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma16_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * 8 * 16 * 4 * (double)iters * blocks * (threads / 32);
    printf("dmma_m16n8k16_tflops %.2f (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  // grid.sync latency
  for (int nb : {sms / 2, sms, 2 * sms}) {
    int iters = 2000; void* args[] = {&iters, &d};
    int maxb = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, gridsync_kernel, 256, 0);
    if (nb > maxb * sms) continue;
    CK(cudaLaunchCooperativeKernel((void*)gridsync_kernel, nb, 256, args, 0, 0)); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)gridsync_kernel, nb, 256, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("grid_sync_us blocks=%d %.3f\n", nb, ms * 1e3 / iters);
  }
  for (int nb : {sms / 2, sms}) {
    int iters = 2000; void* args[] = {&iters, &d};
    unsigned int z = 0;
    CK(cudaMemcpyToSymbol(g_count, &z, 4));
    CK(cudaLaunchCooperativeKernel((void*)flagbar_kernel, nb, 256, args, 0, 0)); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)flagbar_kernel, nb, 256, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("flag_barrier_us blocks=%d %.3f\n", nb, ms * 1e3 / iters);
  }
  // L2-resident read bandwidth
  for (size_t mb : {4, 16, 64}) {
    size_t bytes = mb << 20; double2* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
    int iters = 20; size_t n2 = bytes / 16;
    for (int bl : {sms, sms * 4}) {
      l2read_kernel<<<bl, 512>>>(buf, n2, 2, d); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); l2read_kernel<<<bl, 512>>>(buf, n2, iters, d); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("l2_read_gbs size_mb=%zu blocks=%d %.1f\n", mb, bl, (double)bytes * iters / ms / 1e6);
    }
    cudaFree(buf);
  }
  // DSMEM
  for (int cs : {2, 8, 16}) {
    int words = 8192, iters = 200;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * (sms / cs)); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = words * 8;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (cs > 8) CK(cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, words * 8));
    cudaError_t err = cudaLaunchKernelEx(&cfg, dsmem_kernel, words, 2, d);
    if (err != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) { printf("dsmem cs=%d failed: %s\n", cs, cudaGetErrorString(err)); cudaGetLastError(); continue; }
    cudaEventRecord(e0); CK(cudaLaunchKernelEx(&cfg, dsmem_kernel, words, iters, d)); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double per_sm = (double)words * 8 * iters / (ms * 1e-3) / 1e9;
    printf("dsmem_read_gbs_per_cta cluster=%d %.1f (grid %d)\n", cs, per_sm, cs * (sms / cs));
  }
  // cluster.sync latency
  for (int cs : {8, 16}) {
    int iters = 4000;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * (sms / cs)); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 0;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (cs > 8) CK(cudaFuncSetAttribute(clsync_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaError_t err = cudaLaunchKernelEx(&cfg, clsync_kernel, 10, d);
    if (err != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) { printf("clsync cs=%d failed\n", cs); cudaGetLastError(); continue; }
    cudaEventRecord(e0); CK(cudaLaunchKernelEx(&cfg, clsync_kernel, iters, d)); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("cluster_sync_us cluster=%d %.3f\n", cs, ms * 1e3 / iters);
  }
  // graph node latency
  {
    cudaStream_t s; cudaStreamCreate(&s);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 1000; ++i) empty_kernel<<<sms, 256, 0, s>>>(d);
    cudaStreamEndCapture(s, &g); CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("graph_kernel_node_us %.3f\n", ms * 1e3 / 1000);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 1000; ++i) empty_kernel<<<sms, 256, 0, s>>>(d);
    cudaEventRecord(e1, s); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("stream_kernel_launch_us %.3f\n", ms * 1e3 / 1000);
  }
  printf("done\n");
  return 0;
}
