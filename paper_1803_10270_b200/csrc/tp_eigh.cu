// Batched symmetric eigensolver for the hSVD node Grams (ht.py:346-359:
// eigh(0.5 (G + G^H)), descending, keep <= r_max) on sm_100a: one CTA per k x k
// matrix (k <= 64), the matrix resident in shared memory.
//
//   1. Householder tridiagonalisation A = Q T Q^T (LAPACK dsytd2 order, lower):
//      per column one reflector, p = tau A22 v (4 threads per row), w = p - K v,
//      rank-2 update A22 -= v w^T + w v^T.  ~2/3 k^3 flops and O(k^2) shared
//      traffic per step -- against ~20 k^3 flops and ~3 k^2 shared words per
//      rotation round of the cyclic Jacobi solver it replaces.
//   2. All eigenvalues of T by multisection on Sturm counts (4 lanes per
//      eigenvalue, 5 subintervals per step) to full precision (dstebz).
//   3. Eigenvectors of the nvec largest eigenvalues only (the kept ones) by
//      inverse iteration on T - lambda I (LU with partial pivoting, dstein);
//      eigenvalues closer than 1e-3 ||T|| form clusters whose vectors are
//      re-iterated with modified Gram-Schmidt against the earlier members.
//   4. Back-transformation z <- Q z by the stored reflectors.
// Output as the Jacobi kernels: eigenvalues descending, eigenvector t in column t
// (row-major k x k); columns >= nvec are zero.
#include "tp_common.cuh"
#include <cfloat>

namespace tp {

constexpr int TE_NT = 256;
constexpr int TE_KMAX = 64;

__device__ __forceinline__ int sturm_count(const double* dg, const double* e2, int n, double x, double pivmin) {
  double q = dg[0] - x;
  int c = q < 0.0;
  for (int t = 1; t < n; ++t) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = (dg[t] - x) - e2[t - 1] * rcp_nr(q);   // (<= 1 ulp: the count is backward stable)
    c += q < 0.0;
  }
  return c;
}

// LU with partial pivoting of T - lam I (tridiagonal: diag dg, off-diagonal of); zero
// pivots replaced by eps3 (dlagtf).  u0 holds the reciprocal pivots.
__device__ void tri_factor(const double* dg, const double* of, int n, double lam, double eps3, double* u0, double* u1,
                           double* u2, double* ml, unsigned char* piv) {
  double a = dg[0] - lam;
  double c = n > 1 ? of[0] : 0.0;
  for (int i = 0; i < n - 1; ++i) {
    const double dn = dg[i + 1] - lam, bi = of[i];        // below, next diagonal
    const double cn = (i + 1 < n - 1) ? of[i + 1] : 0.0;  // next super-diagonal
    if (fabs(a) >= fabs(bi)) {   // no interchange
      piv[i] = 0;
      const double ia = rcp_nr((a == 0.0) ? eps3 : a);
      const double m = bi * ia;
      u0[i] = ia; u1[i] = c; u2[i] = 0.0; ml[i] = m;
      a = dn - m * c;
      c = cn;
    } else {                     // swap rows i, i+1
      piv[i] = 1;
      const double m = a * rcp_nr(bi);
      u0[i] = rcp_nr(bi); u1[i] = dn; u2[i] = cn; ml[i] = m;
      a = c - m * dn;
      c = -m * cn;
    }
  }
  u0[n - 1] = rcp_nr((a == 0.0) ? eps3 : a);
}

// solve in place for b with the factors of tri_factor (dlagts)
__device__ void tri_apply(int n, double* b, const double* u0, const double* u1, const double* u2, const double* ml,
                          const unsigned char* piv) {
  for (int i = 0; i < n - 1; ++i) {   // forward: L y = P b
    if (piv[i]) { const double t = b[i]; b[i] = b[i + 1]; b[i + 1] = t; }
    b[i + 1] -= ml[i] * b[i];
  }
  for (int i = n - 1; i >= 0; --i) {   // back: U x = y
    double s = b[i];
    if (i + 1 < n) s -= u1[i] * b[i + 1];
    if (i + 2 < n) s -= u2[i] * b[i + 2];
    b[i] = s * u0[i];
  }
}

__global__ void __launch_bounds__(TE_NT) tridiag_eigh_kernel(int k, int nn, int first, int per, const double* Ain,
                                                             double* Vout, double* wout, int nvec, const int* skip) {
  extern __shared__ double tes[];
  // row stride == 4 (mod 16): the 4-threads-per-row accesses hit distinct banks
  const int n = k, ld = n + (((4 - n % 16) + 16) % 16), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* A = tes;                        // [n][ld]; column j below the subdiagonal keeps reflector j
  double* tau = A + (size_t)n * ld;       // [n]
  double* dg = tau + n;                   // [n] diagonal of T
  double* of = dg + n;                    // [n] off-diagonal of T
  double* e2 = of + n;                    // [n] squared off-diagonal
  double* pv = e2 + n;                    // [n] p
  double* vb = pv + n;                    // [n] current reflector
  double* lam = vb + n;                   // [n] eigenvalues ascending
  double* Z = lam + n;                    // [nvec][n]
  double* scal = Z + (size_t)nvec * n;    // [8]
  const int z = blockIdx.x;
  const size_t base = (size_t)(z / per) * nn + first + z % per;
  if (skip && skip[base]) return;
  const double* in = Ain + base * k * k;
  for (int e = tid; e < n * n; e += TE_NT) {
    const int i = e / n, j = e - i * n;
    A[i * ld + j] = 0.5 * (in[i * k + j] + in[j * k + i]);   // eigh(0.5 (G + G^T)), ht.py:347
  }
  __syncthreads();
  // ---- 1. Householder tridiagonalisation
  // three barriers per reflector: (reflector by warp 0) | p = tau A22 v | rank-2 update;
  // K = tau/2 p.v is formed redundantly by every warp (no barrier)
  for (int j = 0; j + 2 < n; ++j) {
    const int m = n - j - 1;   // length of x = A[j+1 .., j]
    if (warp == 0) {
      double s = 0.0;
      for (int i = 1 + lane; i < m; i += 32) { const double x = A[(j + 1 + i) * ld + j]; s = fma(x, x, s); }
      s = warp_sum(s);
      const double alpha = A[(j + 1) * ld + j];
      double t = 0.0, sc = 0.0, beta = alpha;
      if (s > 0.0) {
        beta = -copysign(sqrt(fma(alpha, alpha, s)), alpha);
        t = (beta - alpha) / beta;
        sc = 1.0 / (alpha - beta);
      }
      if (lane == 0) { tau[j] = t; of[j] = beta; }
      for (int i = lane; i < m; i += 32) {
        const double v = (i == 0) ? 1.0 : A[(j + 1 + i) * ld + j] * sc;
        vb[i] = v;
        if (i > 0) A[(j + 1 + i) * ld + j] = v;
      }
    }
    __syncthreads();
    const double t = tau[j];
    if (t != 0.0) {
      // p = tau A22 v, 4 lanes per row
      {
        const int row = tid >> 2, part = tid & 3;
        double acc = 0.0;
        if (row < m) {
          const double* ar = A + (size_t)(j + 1 + row) * ld + (j + 1);
          for (int c = part; c < m; c += 4) acc = fma(ar[c], vb[c], acc);
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (row < m && part == 0) pv[row] = t * acc;
      }
      __syncthreads();
      double ks = 0.0;
      for (int i = lane; i < m; i += 32) ks = fma(pv[i], vb[i], ks);
      const double K = 0.5 * t * warp_sum(ks);
      {   // rank-2 update, 4 threads per row (no runtime divisions)
        const int row = tid >> 2, part = tid & 3;
        for (int i = row; i < m; i += TE_NT / 4) {
          const double vi = vb[i], wi = pv[i] - K * vi;
          double* ar = A + (size_t)(j + 1 + i) * ld + (j + 1);
          for (int c = part; c < m; c += 4) {
            const double wc = pv[c] - K * vb[c];
            ar[c] = fma(-vi, wc, fma(-wi, vb[c], ar[c]));
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < n; i += TE_NT) {
    dg[i] = A[i * ld + i];
    if (n >= 2 && i == n - 2) of[i] = A[(n - 1) * ld + (n - 2)];
  }
  __syncthreads();
  for (int i = tid; i < n - 1; i += TE_NT) e2[i] = of[i] * of[i];
  if (tid == 0) {
    double lo = INFINITY, hi = -INFINITY, emax = 0.0;
    for (int i = 0; i < n; ++i) {
      const double r = (i > 0 ? fabs(of[i - 1]) : 0.0) + (i < n - 1 ? fabs(of[i]) : 0.0);
      lo = fmin(lo, dg[i] - r);
      hi = fmax(hi, dg[i] + r);
      if (i < n - 1) emax = fmax(emax, of[i] * of[i]);
    }
    const double tn = fmax(fabs(lo), fabs(hi));
    scal[2] = lo - 2.0 * DBL_EPSILON * tn - DBL_MIN;
    scal[3] = hi + 2.0 * DBL_EPSILON * tn + DBL_MIN;
    scal[4] = DBL_MIN * fmax(1.0, emax);   // pivmin (dstebz)
    scal[5] = tn;
  }
  __syncthreads();
  // ---- 2. eigenvalues: multisection, 4 lanes per eigenvalue
  {
    const double pivmin = scal[4];
    // absolute tolerance ~ ulp ||T|| (dstebz's default abstol): what a backward-stable
    // eigensolver resolves; ~22 multisection steps from the Gershgorin interval
    const double atol = 2.0 * DBL_EPSILON * scal[5] + pivmin;
    for (int i0 = 0; i0 < n; i0 += TE_NT / 4) {
      const int idx = i0 + (tid >> 2), part = tid & 3;
      double a = scal[2], b = scal[3];
      for (int it = 0; it < 64; ++it) {
        // warp-uniform exit (the shuffles below need every lane)
        // intervals near zero keep going to relative accuracy: the discarded tail of a
        // rank-deficient Gram is exactly zero in the reference's arithmetic (error estimate)
        const bool done = (b - a <= 2.0 * DBL_EPSILON * fmax(fabs(a), fabs(b)) + pivmin) ||
                          (b - a <= atol && fmin(fabs(a), fabs(b)) > 64.0 * atol);
        if (__all_sync(0xffffffffu, done)) break;
        const double x = a + (double)(part + 1) * (b - a) * 0.2;
        const int c = idx < n ? sturm_count(dg, e2, n, x, pivmin) : 0;
        // new interval: largest x_l with count <= idx, smallest with count > idx
        double na = (c <= idx) ? x : -INFINITY, nb = (c > idx) ? x : INFINITY;
        na = fmax(na, __shfl_xor_sync(0xffffffffu, na, 1));
        na = fmax(na, __shfl_xor_sync(0xffffffffu, na, 2));
        nb = fmin(nb, __shfl_xor_sync(0xffffffffu, nb, 1));
        nb = fmin(nb, __shfl_xor_sync(0xffffffffu, nb, 2));
        if (na > a) a = na;
        if (nb < b) b = nb;
      }
      if (idx < n && part == 0) lam[idx] = 0.5 * (a + b);
    }
  }
  __syncthreads();
  // ---- 3. eigenvectors of the nvec largest eigenvalues (descending t = 0 ..)
  const double tn = scal[5];
  const double eps3 = fmax(DBL_EPSILON * tn, DBL_MIN);
  const double ortol = 1e-3 * tn;
  // shifts (equal eigenvalues perturbed apart, dstein: 10 eps3) and clusters (consecutive
  // kept eigenvalues closer than ortol share a cluster: cs[t] = its first member)
  double* shf = scal + 8;                          // [nvec]
  int* cs = reinterpret_cast<int*>(shf + nvec);    // [nvec]
  if (tid < nvec) {
    const int t = tid;
    double lt = lam[n - 1 - t];
    for (int q = 1; q <= t; ++q)
      if (fabs(lam[n - 1 - t + q] - lt) < 10.0 * eps3) lt -= 10.0 * eps3 * q; else break;
    shf[t] = lt;
    int c0 = t;
    while (c0 > 0 && lam[n - c0] - lam[n - 1 - c0] < ortol) --c0;
    cs[t] = c0;
    double* zt = Z + (size_t)t * n;
    for (int i = 0; i < n; ++i) zt[i] = 1.0 + 0.0625 * (double)((i * 37 + t * 11) % 13) / 13.0;
  }
  __syncthreads();
  // inverse iteration, all kept vectors at once (one thread each), each solve preceded by
  // modified Gram-Schmidt of the cluster members against their earlier members (dstein),
  // done by warp 0 with the vectors spread over the lanes
  double u0[TE_KMAX], u1[TE_KMAX], u2[TE_KMAX], ml[TE_KMAX];   // this thread's LU of T - shift I
  unsigned char piv[TE_KMAX];
  if (tid < nvec) tri_factor(dg, of, n, shf[tid], eps3, u0, u1, u2, ml, piv);
  for (int it = 0; it < 3; ++it) {
    if (warp == 0) {
      for (int t = 1; t < nvec; ++t) {
        double* zs = Z + (size_t)t * n;
        for (int q = cs[t]; q < t; ++q) {
          const double* zq = Z + (size_t)q * n;
          double dot = 0.0, nq = 0.0;
          for (int i = lane; i < n; i += 32) { dot = fma(zq[i], zs[i], dot); nq = fma(zq[i], zq[i], nq); }
          dot = warp_sum(dot);
          nq = warp_sum(nq);
          const double f = nq > 0.0 ? dot / nq : 0.0;
          for (int i = lane; i < n; i += 32) zs[i] = fma(-f, zq[i], zs[i]);
          __syncwarp();
        }
      }
    }
    __syncthreads();
    if (it == 2) break;   // (the last pass only orthogonalises)
    if (tid < nvec) {
      double* zt = Z + (size_t)tid * n;
      tri_apply(n, zt, u0, u1, u2, ml, piv);
      double mx = 0.0;
      for (int i = 0; i < n; ++i) mx = fmax(mx, fabs(zt[i]));
      const double inv = mx > 0.0 ? 1.0 / mx : 1.0;
      for (int i = 0; i < n; ++i) zt[i] *= inv;
    }
    __syncthreads();
  }
  // ---- 4. normalise, back-transform z <- H_0 .. H_{n-3} z (16 lanes per vector)
  for (int v0 = 0; v0 < nvec; v0 += TE_NT / 16) {
    const int t = v0 + (tid >> 4), sl = tid & 15;
    const bool act = t < nvec;
    double* zt = Z + (size_t)(act ? t : 0) * n;
    double s = 0.0;
    if (act)
      for (int i = sl; i < n; i += 16) s = fma(zt[i], zt[i], s);
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
    if (act)
      for (int i = sl; i < n; i += 16) zt[i] *= inv;
    __syncwarp();
    for (int j = n - 3; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      double dot = 0.0;
      if (act)
        for (int i = sl; i < n - j - 1; i += 16) {
          const double v = (i == 0) ? 1.0 : A[(size_t)(j + 1 + i) * ld + j];
          dot = fma(v, zt[j + 1 + i], dot);
        }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (act)
        for (int i = sl; i < n - j - 1; i += 16) {
          const double v = (i == 0) ? 1.0 : A[(size_t)(j + 1 + i) * ld + j];
          zt[j + 1 + i] = fma(-tj * dot, v, zt[j + 1 + i]);
        }
      __syncwarp();
    }
  }
  __syncthreads();
  double* Vo = Vout + base * k * k;
  double* wo = wout + base * k;
  for (int t = tid; t < n; t += TE_NT) wo[t] = lam[n - 1 - t];
  for (int e = tid; e < n * n; e += TE_NT) {
    const int i = e / n, t = e - i * n;
    Vo[i * k + t] = (t < nvec) ? Z[(size_t)t * n + i] : 0.0;
  }
}

size_t tridiag_eigh_smem(int k, int nvec) {
  const size_t ld = (size_t)k + (((4 - k % 16) + 16) % 16);
  return sizeof(double) * ((size_t)k * ld + 7 * (size_t)k + (size_t)nvec * k + 8 + 2 * (size_t)nvec);
}

cudaError_t launch_tridiag_eigh(int nmat, int k, int nn, int first, int per, const double* Ain, double* Vout,
                                double* wout, int nvec, const int* skip, cudaStream_t st) {
  if (k > TE_KMAX || nvec > k) return cudaErrorInvalidValue;
  const size_t smem = tridiag_eigh_smem(k, nvec);
  cudaError_t e = cudaFuncSetAttribute(tridiag_eigh_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tridiag_eigh_kernel<<<nmat, TE_NT, smem, st>>>(k, nn, first, per, Ain, Vout, wout, nvec, skip);
  return cudaGetLastError();
}

}  // namespace tp
