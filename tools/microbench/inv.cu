// Microbenchmark: latency of a 32x32 SPD inversion inside one CTA (cycles), variants:
//  A: warp-register sweep operator (lane = row), rolled pivot loop, selects
//  B: element-parallel sweep, 256 threads, double-buffered smem, 1 barrier/step
//  C: element-parallel sweep, 128 threads (4 warps) with a named barrier
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>

template <int RM>
__device__ void inv_warp(double* A, int r, double* s, double* out) {
  const int lane = threadIdx.x & 31;
  double row[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) row[c] = (lane < r && c < r) ? A[lane * (r + 1) + c] : (c == lane ? 1.0 : 0.0);
  for (int k = 0; k < r; ++k) {
    __syncwarp();
    if (lane == k) {
      double dk = 0.0;
#pragma unroll
      for (int c = 0; c < RM; ++c)
        if (c == k) dk = row[c];
      const double id = 1.0 / dk;
#pragma unroll
      for (int c = 0; c < RM; ++c) s[c] = (c == k) ? -id : row[c] * id;
      s[RM] = dk;
    }
    __syncwarp();
    const double dk = s[RM];
    if (lane != k) {
      const double sk = s[lane];
      const double f = sk * dk;
#pragma unroll
      for (int c = 0; c < RM; ++c) row[c] = (c == k) ? sk : fma(-f, s[c], row[c]);
    } else {
#pragma unroll
      for (int c = 0; c < RM; ++c) row[c] = s[c];
    }
  }
  if (lane < r)
#pragma unroll
    for (int c = 0; c < RM; ++c)
      if (c < r) out[lane * (r + 1) + c] = -row[c];
}

// element-parallel sweep: nthr threads own r*r/nthr elements each; buffers B0/B1 (r x (r+1))
template <int NT>
__device__ void inv_par(double* B0, double* B1, int r, int t, int bar_id) {
  const int rp = r + 1;
  double* src = B0;
  double* dst = B1;
  for (int k = 0; k < r; ++k) {
    const double d = src[k * rp + k];
    const double id = 1.0 / d;
    for (int e = t; e < r * r; e += NT) {
      const int i = e / r, c = e - i * r;
      const double aik = src[i * rp + k], akc = src[k * rp + c];
      double v;
      if (i == k && c == k) v = -id;
      else if (i == k) v = akc * id;
      else if (c == k) v = aik * id;
      else v = fma(-aik * id, akc, src[i * rp + c]);
      dst[i * rp + c] = v;
    }
    if (NT == 256) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(NT));
    double* tmp = src; src = dst; dst = tmp;
  }
  if (r & 1) {  // result in B1 after odd steps: copy back to B0
    for (int e = t; e < r * r; e += NT) {
      const int i = e / r, c = e - i * r;
      B0[i * rp + c] = B1[i * rp + c];
    }
  }
}

// fast reciprocal: MUFU seed + 2 Newton steps (<= 1 ulp, no slow path)
__device__ __forceinline__ double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}

// element-parallel symmetric sweep with the elements in registers.
// NT threads; thread t owns row i = t / TPR, columns c = (t % TPR) + TPR*u, u < EPT.
// Only the pivot row is published per step (symmetry: column k == row k).
template <int NT, int EPT>
__device__ void inv_reg(const double* A, int r, double* pub /* 2 x 32 */, double* out, int bar_id) {
  constexpr int TPR = 32 / EPT;           // threads per row (r <= 32)
  const int t = threadIdx.x;
  const int i = t / TPR, c0 = t % TPR;
  const int rp = r + 1;
  double v[EPT];
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int c = c0 + TPR * u;
    v[u] = (i < r && c < r) ? A[i * rp + c] : 0.0;
  }
  // publish row 0
  if (i == 0)
#pragma unroll
    for (int u = 0; u < EPT; ++u) pub[c0 + TPR * u] = v[u];
  if (NT == 256) __syncthreads(); else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(NT));
  for (int k = 0; k < r; ++k) {
    const double* rk = pub + (k & 1) * 32;
    double* rn = pub + ((k + 1) & 1) * 32;
    const double d = rk[k];
    const double id = rcp_nr(d);
    const double aik = (i < r) ? rk[i] : 0.0;   // column k == row k
    const double f = aik * id;
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + TPR * u;
      const double akc = rk[c];
      double nv = fma(-f, akc, v[u]);
      nv = (c == k) ? f : nv;
      nv = (i == k) ? ((c == k) ? -id : akc * id) : nv;
      v[u] = nv;
    }
    if (i == k + 1)
#pragma unroll
      for (int u = 0; u < EPT; ++u) rn[c0 + TPR * u] = v[u];
    if (NT == 256) __syncthreads(); else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(NT));
  }
  if (i < r)
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + TPR * u;
      if (c < r) out[i * rp + c] = -v[u];
    }
}

// 2x2-block symmetric sweep: pivot pairs (2m, 2m+1); elements in registers;
// rows p, q published per block step (symmetry gives the pivot columns)
template <int NT, int EPT>
__device__ void inv_reg2(const double* A, int r, double* pub /* 2 x 2 x 32 */, double* out, int bar_id) {
  constexpr int TPR = 32 / EPT;
  const int t = threadIdx.x;
  const int i = t / TPR, c0 = t % TPR;
  const int rp = r + 1;
  double v[EPT];
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int c = c0 + TPR * u;
    v[u] = (i < r && c < r) ? A[i * rp + c] : ((i == c) ? 1.0 : 0.0);   // identity padding to 32
  }
  if (i < 2)
#pragma unroll
    for (int u = 0; u < EPT; ++u) pub[i * 32 + c0 + TPR * u] = v[u];
  if (NT == 256) __syncthreads(); else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(NT));
  const int rr = (r + 1) & ~1;
  for (int k = 0; k < rr; k += 2) {
    const double* Rp = pub + ((k >> 1) & 1) * 64;
    const double* Rq = Rp + 32;
    double* Np = pub + (((k >> 1) + 1) & 1) * 64;
    const double a = Rp[k], b = Rp[k + 1], cc = Rq[k + 1];
    const double idet = rcp_nr(fma(a, cc, -b * b));
    const double p00 = cc * idet, p01 = -b * idet, p11 = a * idet;      // P^-1
    const double xi = Rp[i], yi = Rq[i];                                // (A_ip, A_iq)
    const double ti0 = xi * p00 + yi * p01, ti1 = xi * p01 + yi * p11;  // (A_iK P^-1)
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + TPR * u;
      const double rc0 = Rp[c], rc1 = Rq[c];
      const double w0 = p00 * rc0 + p01 * rc1, w1 = p01 * rc0 + p11 * rc1;   // P^-1 A_Kc
      double nv = fma(-xi, w0, fma(-yi, w1, v[u]));
      const bool ck = (c == k) || (c == k + 1), ik = (i == k) || (i == k + 1);
      if (ck) nv = (c == k) ? ti0 : ti1;
      if (ik) nv = (i == k) ? w0 : w1;
      if (ik && ck) nv = -((i == k) ? ((c == k) ? p00 : p01) : ((c == k) ? p01 : p11));
      v[u] = nv;
    }
    if (i == k + 2 || i == k + 3)
#pragma unroll
      for (int u = 0; u < EPT; ++u) Np[(i - k - 2) * 32 + c0 + TPR * u] = v[u];
    if (NT == 256) __syncthreads(); else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(NT));
  }
  if (i < r)
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + TPR * u;
      if (c < r) out[i * rp + c] = -v[u];
    }
}

__global__ void bench(const double* Ain, int r, int reps, int variant, long long* cyc, double* out) {
  __shared__ double A[33 * 33], B0[33 * 33], B1[33 * 33], s[160];
  for (int e = threadIdx.x; e < r * (r + 1); e += blockDim.x) A[e] = Ain[e];
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < reps; ++it) {
    if (variant == 0) {
      if (threadIdx.x < 32) inv_warp<32>(A, r, s, B0);
      __syncthreads();
    } else if (variant == 1) {
      for (int e = threadIdx.x; e < r * (r + 1); e += 256) B0[e] = A[e];
      __syncthreads();
      inv_par<256>(B0, B1, r, threadIdx.x, 0);
      __syncthreads();
    } else if (variant == 3) {
      if (threadIdx.x < 128) inv_reg<128, 8>(A, r, s, B0, 1);
      __syncthreads();
    } else if (variant == 4) {
      inv_reg<256, 4>(A, r, s, B0, 0);
      __syncthreads();
    } else if (variant == 6) {
      inv_reg2<256, 4>(A, r, s, B0, 0);
      __syncthreads();
    } else if (variant == 5) {
      if (threadIdx.x < 64) inv_reg<64, 16>(A, r, s, B0, 1);
      __syncthreads();
    } else {
      if (threadIdx.x < 128) {
        for (int e = threadIdx.x; e < r * (r + 1); e += 128) B0[e] = A[e];
        asm volatile("bar.sync 1, 128;");
        inv_par<128>(B0, B1, r, threadIdx.x, 1);
      }
      __syncthreads();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
  for (int e = threadIdx.x; e < r * (r + 1); e += blockDim.x) out[e] = (variant == 0 || variant >= 3) ? B0[e] : -B0[e];
}

int main() {
  const int r = 32, rp = 33;
  double h[33 * 33];
  srand(1);
  // SPD: M M^T + r I
  double M[32][32];
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) M[i][j] = (double)rand() / RAND_MAX - 0.5;
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      double v = (i == j) ? r : 0.0;
      for (int k = 0; k < r; ++k) v += M[i][k] * M[j][k];
      h[i * rp + j] = v;
    }
  double *dA, *dout;
  long long* dc;
  cudaMalloc(&dA, sizeof(h));
  cudaMalloc(&dout, sizeof(h));
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int v = 3; v < 7; ++v) {
    bench<<<1, 256>>>(dA, r, 2, v, dc, dout);
    bench<<<1, 256>>>(dA, r, 20, v, dc, dout);
    long long c;
    double o[33 * 33];
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
    // check A * Ainv = I
    double err = 0;
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < r; ++j) {
        double acc = 0;
        for (int k = 0; k < r; ++k) acc += h[i * rp + k] * o[k * rp + j];
        err = fmax(err, fabs(acc - (i == j)));
      }
    printf("variant %d: %lld cycles per 32x32 inversion, |A Ainv - I| = %.2e  (%s)\n", v, c, err,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
