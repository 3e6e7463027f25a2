// Split timing of had / Y DMMA / Y stores (copy of cl_had_y with phase switches)
#include <cstdio>
#include "../../paper_1803_10270_b200/csrc/tp_als.cu"
namespace tp {
int inner_tiles(int, int, int) { return 1; }
int launch_inner(int, const int*, int, const double*, int, const double*, int, double*, double*, cudaStream_t) { return 0; }
void set_last_error(cudaError_t) {}
int cuda_status(cudaError_t e) { return e == cudaSuccess ? 0 : -1; }
}
using namespace tp;

template <int RM, int MODE>   // bit0 had, bit1 Y dmma, bit2 stores
__device__ void hy(const AlsArgs& a, const Smem& sm, int j, int w, int b, int cid, int Pr) {
  constexpr int NT = RM / 8;
  const int r = a.r, rh = pad4(r), ldw = a.ldw, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cs32 = smem_u32(sm.Cs), ks = 8u * (uint32_t)(r * a.wmax);
  if (MODE & 1) {
    for (int e = tid; e < r * w; e += ALS_NT) {
      const int l = e / w, c = e - l * w;
      const uint32_t base = cs32 + 8u * (uint32_t)(l * a.wmax + c);
      double f[TP_MAXD];
#pragma unroll
      for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < a.d && k != j) ? lds64(base + (uint32_t)k * ks) : 1.0;
      double v = 1.0;
#pragma unroll
      for (int k = 0; k < TP_MAXD; ++k) v *= f[k];
      sm.hadT[c * rh + l] = v;
    }
    __syncthreads();
  }
  const int Qj = a.q[j], Pq = a.Pq, qb0 = Qj * b / Pq, nb = Qj * (b + 1) / Pq - qb0;
  const int mt = (nb + 7) / 8, kst = (w + 3) / 4;
  const uint32_t vs32 = smem_u32(sm.Vs + a.qoffc[j]), hd32 = smem_u32(sm.hadT);
  for (int m = warp; m < mt; m += ALS_NW) {
    const int s = m * 8 + (lane >> 2);
    const uint32_t arow = vs32 + 8u * (uint32_t)(s * ldw + (lane & 3));
    const uint32_t brow = hd32 + 8u * (uint32_t)((lane & 3) * rh + (lane >> 2));
    double acc[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = (double)s;
    if (MODE & 2) {
#pragma unroll 2
      for (int kk = 0; kk < kst; ++kk) {
        const double av = lds64(arow + 32u * (uint32_t)kk);
        double fb[NT];
#pragma unroll
        for (int n = 0; n < NT; ++n) fb[n] = lds64(brow + 8u * (uint32_t)(4 * kk * rh + 8 * n));
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[n][0], acc[n][1], av, fb[n]);
      }
    }
    if ((MODE & 4) && s < nb) {
      const int rm = sm.rowmap[j * a.qmax + qb0 + s];
      const int pc = rm >> 16, ii = rm & 0xffff;
      double* yrow = a.Y + (((size_t)pc * Pr + cid) * a.ncolmax + ii) * r;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int ocol = n * 8 + 2 * (lane & 3);
        *reinterpret_cast<double2*>(yrow + ocol) = make_double2(acc[n][0], acc[n][1]);
      }
    } else if (acc[0][0] == 1234.5) {
      sm.rb[0] = acc[0][1] + acc[1][0] + acc[2][0] + acc[3][1];
    }
  }
}

template <int MODE>
__global__ void bench(AlsArgs a, int w, int reps, long long* cyc) {
  extern __shared__ double smem[];
  const Smem sm = carve_cl(smem, a, 33);
  for (int e = threadIdx.x; e < a.sumqs * a.ldw; e += 256) sm.Vs[e] = 1e-3 * (e % 89);
  for (int e = threadIdx.x; e < 6 * 32 * a.wmax; e += 256) sm.Cs[e] = 1.0 + 1e-3 * (e % 7);
  for (int e = threadIdx.x; e < 6 * 256; e += 256) sm.rowmap[e] = ((e % 256) / 2 << 16) | (e & 1);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) { hy<32, MODE>(a, sm, 1, w, 0, 0, 33); __syncthreads(); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[MODE] = (t1 - t0) / reps;
}

int main() {
  AlsArgs a;
  memset(&a, 0, sizeof(a));
  const int d = 6, r = 32, w = 16, Pq = 4, nb = 64;
  a.d = d; a.r = r; a.R = 512; a.Pq = Pq; a.wmax = w; a.ldw = pad4(w); a.nbmax = nb; a.sumqs = d * nb + 8;
  a.ncolmax = 2; a.qmax = 256;
  a.chunk = 200;
  for (int k = 0; k < d; ++k) { a.q[k] = 256; a.qoffc[k] = k * nb * a.ldw; }
  size_t smem = cl_smem_doubles(d, r, w, a.ldw, a.sumqs, nb, a.ncolmax, 33, Pq, a.chunk, 256) * 8;
  long long* c; cudaMalloc(&c, 64 * 8);
  double* Y; cudaMalloc(&Y, 1 << 24); a.Y = Y;
#define RUN(M) cudaFuncSetAttribute(bench<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
  bench<M><<<1, 256, smem>>>(a, w, 20, c); bench<M><<<1, 256, smem>>>(a, w, 20, c);
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(6) RUN(7)
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  printf("%s: none %lld | had %lld | dmma %lld | had+dmma %lld | stores %lld | dmma+stores %lld | all %lld\n",
         cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[6], h[7]);
  return 0;
}
