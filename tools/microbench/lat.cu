// Dependent-chain latencies (cycles) on sm_100a: DFMA, DADD, LDS.64, DMMA m8n8k4, shfl f64, bar.sync
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k(double* io, long long* cyc, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)((i * 7 + 3) & 1023) ;
  __syncthreads();
  double x = io[threadIdx.x], y = io[threadIdx.x + 32];
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, y, 1.0); x = fma(x, y, 1.0); x = fma(x, y, 1.0); x = fma(x, y, 1.0); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / (4 * n);
  t0 = clock64();
  int idx = threadIdx.x & 1023;
  for (int i = 0; i < n; ++i) { idx = (int)s[idx]; idx = (int)s[idx]; idx = (int)s[idx]; idx = (int)s[idx]; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / (4 * n);
  double c0 = 0, c1 = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(x), "d"(y));
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / (4 * n);
  t0 = clock64();
  for (int i = 0; i < n; ++i) { y = __shfl_xor_sync(0xffffffffu, y, 1); y = __shfl_xor_sync(0xffffffffu, y, 2); y = __shfl_xor_sync(0xffffffffu, y, 4); y = __shfl_xor_sync(0xffffffffu, y, 8); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / (4 * n);
  t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / (4 * n);
  // 8 independent DMMA chains per warp: throughput per warp
  double d[8][2] = {};
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[u][0]), "+d"(d[u][1]) : "d"(x), "d"(y));
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / (8 * n);
  double acc = 0; for (int u = 0; u < 8; ++u) acc += d[u][0] + d[u][1];
  io[threadIdx.x] = x + c0 + c1 + idx + acc;
}
int main() {
  double* io; long long* c; cudaMalloc(&io, 4096 * 8); cudaMalloc(&c, 64 * 8);
  cudaMemset(io, 0, 4096 * 8);
  long long h[8];
  for (int bs : {32, 256}) {
    k<<<1, bs>>>(io, c, 1000); k<<<1, bs>>>(io, c, 1000);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("block %d: DFMA dep %lld, LDS dep %lld, DMMA dep %lld, SHFL dep %lld, DADD dep %lld, DMMA 8-chain/warp interval %lld\n",
           bs, h[0], h[1], h[2], h[3], h[4], h[5]);
  }
  return 0;
}
