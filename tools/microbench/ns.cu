// Microbenchmark (one CTA, 256 threads): latency in cycles of the pieces of the
// ALS mode inverse: DMMA 32x32x32 small GEMM at smem stride 33 vs 36, block max,
// build of A, and one Newton-Schulz step.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_runtime.h>
#include <cstdio>
#include <cmath>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma_v(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// C = I - A B (mode 0) for 32x32 at stride LD; 8 warps x 2 tiles, K split in SPLIT chains
template <int LD, bool VOL>
__device__ void gemm32(const double* A, const double* B, double* C) {
  constexpr int TPW = 2, KS = 8, SPLIT = 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[TPW][SPLIT][2];
#pragma unroll
  for (int t = 0; t < TPW; ++t)
#pragma unroll
    for (int s = 0; s < SPLIT; ++s) acc[t][s][0] = acc[t][s][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int k = 4 * kk + (lane & 3);
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int tile = warp + t * 8;
      const int m0 = (tile >> 2) * 8, n0 = (tile & 3) * 8;
      const double fa = A[(m0 + (lane >> 2)) * LD + k];
      const double fb = B[k * LD + n0 + (lane >> 2)];
      if (VOL) dmma_v(acc[t][kk % SPLIT][0], acc[t][kk % SPLIT][1], fa, fb);
      else dmma(acc[t][kk % SPLIT][0], acc[t][kk % SPLIT][1], fa, fb);
    }
  }
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int tile = warp + t * 8;
    double s0 = acc[t][0][0], s1 = acc[t][0][1];
#pragma unroll
    for (int s = 1; s < SPLIT; ++s) { s0 += acc[t][s][0]; s1 += acc[t][s][1]; }
    const int orow = (tile >> 2) * 8 + (lane >> 2), oc = (tile & 3) * 8 + 2 * (lane & 3);
    C[orow * LD + oc] = (orow == oc ? 1.0 : 0.0) - s0;
    C[orow * LD + oc + 1] = (orow == oc + 1 ? 1.0 : 0.0) - s1;
  }
}

template <int LD>
__device__ double bmax(const double* M, double* red) {
  double m = 0.0;
  for (int e = threadIdx.x; e < 1024; e += 256) m = fmax(m, fabs(M[(e >> 5) * LD + (e & 31)]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  double out = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) out = fmax(out, red[w]);
  __syncthreads();
  return out;
}

__global__ void bench(const double* Ain, int reps, long long* cyc, double* sink) {
  __shared__ double A[32 * 36], X[32 * 36], Rm[32 * 36], red[16], Gs[2 * 1024];
  for (int e = threadIdx.x; e < 32 * 36; e += 256) { A[e] = Ain[e % 1024]; X[e] = Ain[(e * 7) % 1024]; }
  for (int e = threadIdx.x; e < 2 * 1024; e += 256) Gs[e] = Ain[e % 1024];
  __syncthreads();
  double acc = 0.0;
  long long t0, t1;
#define TIME(slot, ...)                                           \
  __syncthreads();                                                 \
  acc += *(volatile double*)red;                                   \
  t0 = clock64();                                                  \
  for (int it = 0; it < reps; ++it) { __VA_ARGS__; __syncthreads(); acc += *(volatile double*)(Rm + threadIdx.x); } \
  t1 = clock64();                                                  \
  if (threadIdx.x == 0) cyc[slot] = (t1 - t0) / reps;
  TIME(0, gemm32<33, true>(A, X, Rm));
  TIME(1, gemm32<33, false>(A, X, Rm));
  TIME(2, gemm32<36, true>(A, X, Rm));
  TIME(3, gemm32<36, false>(A, X, Rm));
  TIME(4, acc += bmax<36>(Rm, red));
  TIME(5, {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      double v = 1.0;
      for (int k = 0; k < 6; ++k) if (k != 2) v *= Gs[(k % 2) * 1024 + e];
      A[(e >> 5) * 36 + (e & 31)] = v;
    }
  });
  TIME(6, {});
  if (threadIdx.x == 0) *sink = acc;
}

int main() {
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = (i % 33 == 0) ? 2.0 : 0.001 * ((i * 37) % 11);
  double *d, *sink; long long* c;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&sink, 8); cudaMalloc(&c, 16 * 8);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  bench<<<1, 256>>>(d, 100, c, sink);
  bench<<<1, 256>>>(d, 100, c, sink);
  long long hc[16];
  cudaMemcpy(hc, c, sizeof(hc), cudaMemcpyDeviceToHost);
  const char* nm[] = {"gemm32 ld33 volatile", "gemm32 ld33", "gemm32 ld36 volatile", "gemm32 ld36", "block max",
                      "build A (5 Hadamard)", "empty (sync + load)"};
  for (int i = 0; i < 7; ++i) printf("%-24s %6lld cycles\n", nm[i], hc[i]);
  return 0;
}
