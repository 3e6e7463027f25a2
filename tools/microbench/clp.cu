// Standalone cost (cycles, one CTA) of the ALS cluster-variant phases, using the
#include <cstdio>
// kernel's own device code: cl_partials (cross + Gram partial GEMM), had + Y.
#include "../../paper_1803_10270_b200/csrc/tp_als.cu"
namespace tp {
int inner_tiles(int, int, int) { return 1; }
int launch_inner(int, const int*, int, const double*, int, const double*, int, double*, double*, cudaStream_t) { return 0; }
void set_last_error(cudaError_t) {}
int cuda_status(cudaError_t e) { return e == cudaSuccess ? 0 : -1; }
}
using namespace tp;

__global__ void bench(AlsArgs a, int w, int nb, int reps, long long* cyc) {
  extern __shared__ double smem[];
  const int Pr = 33;
  const Smem sm = carve_cl(smem, a, Pr);
  for (int e = threadIdx.x; e < 64 * 36; e += 256) sm.Us[e] = 1e-3 * (e % 97);
  for (int e = threadIdx.x; e < a.sumqs * a.ldw; e += 256) sm.Vs[e] = 1e-3 * (e % 89);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) cl_partials<32>(a, sm, 0, w, nb, 0, 33);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
  for (int e = threadIdx.x; e < 6 * 32 * a.wmax; e += 256) sm.Cs[e] = 1.0 + 1e-3 * (e % 7);
  for (int e = threadIdx.x; e < 6 * 256; e += 256) sm.rowmap[e] = ((e % 256) / 2 << 16) | (e & 1);
  __syncthreads();
  t0 = clock64();
  for (int it = 0; it < reps; ++it) { cl_had_y<32>(a, sm, 1, w, 0, 0, Pr); __syncthreads(); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / reps;
}

int main() {
  AlsArgs a;
  memset(&a, 0, sizeof(a));
  const int d = 6, r = 32, w = 16, Pq = 4, nb = 64;
  a.d = d; a.r = r; a.R = 512; a.Pq = Pq; a.wmax = w; a.ldw = pad4(w); a.nbmax = nb; a.sumqs = d * nb + 8;
  a.ncolmax = 2; a.qmax = 256;
  a.chunk = (r * w + r * r + Pq - 1) / Pq; a.chunk += a.chunk & 1;
  for (int k = 0; k < d; ++k) { a.q[k] = 256; a.qoffc[k] = k * nb * a.ldw; }
  size_t smem = cl_smem_doubles(d, r, w, a.ldw, a.sumqs, nb, a.ncolmax, 33, Pq, a.chunk, 256) * 8;
  printf("smem %zu\n", smem);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  long long* c; cudaMalloc(&c, 64);
  double* Y; cudaMalloc(&Y, 1 << 24); a.Y = Y;
  bench<<<1, 256, smem>>>(a, w, nb, 20, c);
  bench<<<1, 256, smem>>>(a, w, nb, 20, c);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("%s: cl_partials (r=32, w=16, nb=64): %lld cycles, had+Y %lld cycles\n", cudaGetErrorString(e), h[0], h[1]);
  return 0;
}
