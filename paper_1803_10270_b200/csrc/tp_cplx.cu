// Complex128 CP path for sm_100a: the reference's own
// arithmetic (cp.py coerces every factor to complex128, cp.py:59; the Fourier
// Galerkin basis has complex factor matrices, basis.py:168-187), so the
// reference's experiments and rank_reduce_als with its complex random terms
// (cp.py:129-136, 356-360) run on the GPU unchanged.
//
// Complex numbers are interleaved (re, im) fp64 pairs, the memory layout of
// numpy / torch complex128.  Kernels:
//   cp_apply_c_kernel  -- operators.apply (operators.py:48-62) with complex
//                         weights / factor matrices, term-major, weight in mode 0
//   cp_inner_c_kernel  -- <f, g> = sum_{l,n} prod_k (F_k^H G_k)[l, n] (cp.py:111-121),
//                         fixed-order two-pass reduction (deterministic)
//   als_c_kernel       -- cp_approx_als (cp.py:266-334) for problems that fit one
//                         CTA's shared memory (the reference's experiments: d <= 6,
//                         Q <= ~100, ranks <= 32): crosses, Grams, Hadamards,
//                         right-hand sides, the complex Gauss-Jordan inverse of the
//                         Hermitian normal matrix, the residual trace and the
//                         stopping rules, all resident.
#include "tp_common.cuh"
#include <cmath>
#include <cstring>

namespace tp {

struct cplx {
  double x, y;
};
__device__ __forceinline__ cplx cmk(double a, double b) { cplx c; c.x = a; c.y = b; return c; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
// acc + conj(a) b
__device__ __forceinline__ cplx cfma_conj(cplx a, cplx b, cplx acc) {
  return cmk(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}
// acc + a b
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx acc) {
  return cmk(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
__device__ __forceinline__ cplx crcp(cplx a) {
  const double s = 1.0 / fma(a.x, a.x, a.y * a.y);
  return cmk(a.x * s, -a.y * s);
}
__device__ __forceinline__ cplx ld(const double* p, size_t i) { return cmk(p[2 * i], p[2 * i + 1]); }
__device__ __forceinline__ void st(double* p, size_t i, cplx v) { p[2 * i] = v.x; p[2 * i + 1] = v.y; }

// ---------------------------------------------------------------------------
// operator apply (complex)
// ---------------------------------------------------------------------------
constexpr int APC_MAXT = 64;

struct ApplyCArgs {
  int d, r_in, R_out, col_off, n_terms;
  int q[TP_MAXD];
  long long offF[TP_MAXD], offO[TP_MAXD];   // complex element offsets
  const double* F;
  double* out;
  const double* mats;
  double w0[2 * APC_MAXT];                   // scale * weight per term (mode 0)
  long long moff[APC_MAXT][TP_MAXD];         // complex element offset of the matrix, -1 = identity
};

__global__ void __launch_bounds__(256) cp_apply_c_kernel(const __grid_constant__ ApplyCArgs a) {
  const int t = blockIdx.x, k = blockIdx.y;
  const int Q = a.q[k], r = a.r_in;
  const double* Fk = a.F + 2 * a.offF[k];
  double* Ok = a.out + 2 * a.offO[k];
  const long long mo = a.moff[t][k];
  const cplx sc = (k == 0) ? cmk(a.w0[2 * t], a.w0[2 * t + 1]) : cmk(1.0, 0.0);
  const int col = a.col_off + t * r;
  for (int e = blockIdx.z * blockDim.x + threadIdx.x; e < Q * r; e += gridDim.z * blockDim.x) {
    const int s = e / r, c = e % r;
    cplx v;
    if (mo < 0) {
      v = ld(Fk, (size_t)s * r + c);
    } else {
      const double* E = a.mats + 2 * (mo + (long long)s * Q);
      v = cmk(0.0, 0.0);
      for (int u = 0; u < Q; ++u) v = cfma(ld(E, u), ld(Fk, (size_t)u * r + c), v);
    }
    st(Ok, (size_t)s * a.R_out + col + c, cmul(sc, v));
  }
}

// ---------------------------------------------------------------------------
// inner product (complex): partial[l * rb + n] = prod_k sum_s conj(A_k[s,l]) B_k[s,n],
// then one CTA sums the partials in a fixed order
// ---------------------------------------------------------------------------
struct QOffC { int q[TP_MAXD]; long long oa[TP_MAXD], ob[TP_MAXD]; };

__global__ void __launch_bounds__(256) cp_inner_c_kernel(int d, QOffC qo, int ra, const double* A, int rb,
                                                         const double* B, double* part) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)ra * rb) return;
  const int l = (int)(e / rb), n = (int)(e % rb);
  cplx prod = cmk(1.0, 0.0);
  for (int k = 0; k < d; ++k) {
    const double* Ak = A + 2 * qo.oa[k];
    const double* Bk = B + 2 * qo.ob[k];
    cplx acc = cmk(0.0, 0.0);
    for (int s = 0; s < qo.q[k]; ++s) acc = cfma_conj(ld(Ak, (size_t)s * ra + l), ld(Bk, (size_t)s * rb + n), acc);
    prod = cmul(prod, acc);
  }
  st(part, e, prod);
}

__global__ void __launch_bounds__(256) sum_c_kernel(const double* part, long long n, double* out) {
  __shared__ double rx[256], ry[256];
  double sx = 0.0, sy = 0.0;
  for (long long e = threadIdx.x; e < n; e += 256) { sx += part[2 * e]; sy += part[2 * e + 1]; }
  rx[threadIdx.x] = sx; ry[threadIdx.x] = sy;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) { rx[threadIdx.x] += rx[threadIdx.x + w]; ry[threadIdx.x] += ry[threadIdx.x + w]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = rx[0]; out[1] = ry[0]; }
}

static int launch_inner_c(int d, const int* q, int ra, const double* A, int rb, const double* B, double* out,
                          double* part, cudaStream_t st) {
  QOffC qo;
  memset(&qo, 0, sizeof(qo));
  long long oa = 0, ob = 0;
  for (int k = 0; k < d; ++k) {
    qo.q[k] = q[k]; qo.oa[k] = oa; qo.ob[k] = ob;
    oa += (long long)q[k] * ra; ob += (long long)q[k] * rb;
  }
  const long long n = (long long)ra * rb;
  cp_inner_c_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d, qo, ra, A, rb, B, part);
  sum_c_kernel<<<1, 256, 0, st>>>(part, n, out);
  return cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// fused complex ALS, one CTA
// ---------------------------------------------------------------------------
constexpr int ALSC_NT = 256;

struct AlsCArgs {
  int d, R, r, sweeps, qmax, sumq;
  int q[TP_MAXD], qo[TP_MAXD];
  const double* V;
  double* U;
  const double* norm_sq;   // [2] <V, V> (real part used)
  double* trace;
  int* info;
  double reg;
  int reg_mode;
  double tol, stall;
  int need_resid;
};

__host__ __device__ inline size_t als_c_smem_doubles(int d, int sumq, int qmax, int R, int r) {
  // complex counts: V sumq*R, U sumq*r, C d*r*R, G d*r*r, had r*R, rhs r*qmax, Ai r*r, rowk r, colk r
  const size_t c = (size_t)sumq * R + (size_t)sumq * r + (size_t)d * r * R + (size_t)d * r * r + (size_t)r * R +
                   (size_t)r * qmax + (size_t)r * r + 2 * (size_t)r;
  return 2 * c + 2 * ALSC_NT + 8;
}

__device__ inline double blk_sum_c(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = ALSC_NT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

__global__ void __launch_bounds__(ALSC_NT, 1) als_c_kernel(const __grid_constant__ AlsCArgs a) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, d = a.d, R = a.R, r = a.r, rr = r * r;
  double* Vs = sm;                                   // [sumq][R]
  double* Us = Vs + 2 * (size_t)a.sumq * R;          // [sumq][r]
  double* Cs = Us + 2 * (size_t)a.sumq * r;          // [d][r][R]  C_k = U_k^H V_k
  double* Gs = Cs + 2 * (size_t)d * r * R;           // [d][r][r]  G_k = U_k^H U_k
  double* had = Gs + 2 * (size_t)d * rr;             // [r][R]
  double* rhs = had + 2 * (size_t)r * R;             // [r][qmax]
  double* Ai = rhs + 2 * (size_t)r * a.qmax;         // [r][r]
  double* rowk = Ai + 2 * (size_t)rr;                // [r]
  double* colk = rowk + 2 * (size_t)r;               // [r]
  double* red = colk + 2 * (size_t)r;                // [ALSC_NT]
  double* red2 = red + ALSC_NT;                      // [ALSC_NT]
  for (size_t e = tid; e < 2 * (size_t)a.sumq * R; e += ALSC_NT) Vs[e] = a.V[e];
  for (size_t e = tid; e < 2 * (size_t)a.sumq * r; e += ALSC_NT) Us[e] = a.U[e];
  __syncthreads();
  auto refresh = [&](int k) {   // C_k, G_k from U_k (cp.py:190-195, 318-320)
    const double* Uk = Us + 2 * (size_t)a.qo[k] * r;
    const double* Vk = Vs + 2 * (size_t)a.qo[k] * R;
    const int Q = a.q[k], n1 = r * R;
    for (int o = tid; o < n1 + rr; o += ALSC_NT) {
      cplx acc = cmk(0.0, 0.0);
      if (o < n1) {
        const int l = o / R, c = o - l * R;
        for (int s = 0; s < Q; ++s) acc = cfma_conj(ld(Uk, (size_t)s * r + l), ld(Vk, (size_t)s * R + c), acc);
        st(Cs, (size_t)k * n1 + o, acc);
      } else {
        const int g = o - n1, l = g / r, m = g - l * r;
        for (int s = 0; s < Q; ++s) acc = cfma_conj(ld(Uk, (size_t)s * r + l), ld(Uk, (size_t)s * r + m), acc);
        st(Gs, (size_t)k * rr + g, acc);
      }
    }
  };
  for (int k = 0; k < d; ++k) refresh(k);
  __syncthreads();
  const double norm_sq = a.need_resid ? fmax(a.norm_sq[0], 0.0) : 0.0;
  const double t_norm = sqrt(norm_sq);
  double prev = INFINITY;
  int status = 0, done = 0;
  for (int sweep = 0; sweep < a.sweeps; ++sweep) {
    for (int j = 0; j < d; ++j) {
      const int Qj = a.q[j];
      // Hadamards of the crosses (cp.py:197-201) and of the Grams (cp.py:312-315) + lambda I
      for (int e = tid; e < r * R; e += ALSC_NT) {
        cplx v = cmk(1.0, 0.0);
        for (int k = 0; k < d; ++k)
          if (k != j) v = cmul(v, ld(Cs, (size_t)k * r * R + e));
        st(had, e, v);
      }
      for (int e = tid; e < rr; e += ALSC_NT) {
        cplx v = cmk(1.0, 0.0);
        for (int k = 0; k < d; ++k)
          if (k != j) v = cmul(v, ld(Gs, (size_t)k * rr + e));
        st(Ai, e, v);
      }
      __syncthreads();
      double lam = a.reg;
      if (a.reg_mode) {   // lambda = reg * max(Re tr A, 0) / r  (cp.py:172)
        double tr = 0.0;
        for (int i = 0; i < r; ++i) tr += Ai[2 * ((size_t)i * r + i)];
        lam = a.reg * fmax(tr, 0.0) / (double)r;
        __syncthreads();   // every thread has read the diagonal
      }
      if (tid < r) Ai[2 * ((size_t)tid * r + tid)] += lam;
      // rhs[l][s] = sum_c had[l][c] V_j[s][c]  (had @ T_j^T, cp.py:203)
      const double* Vj = Vs + 2 * (size_t)a.qo[j] * R;
      for (int o = tid; o < r * Qj; o += ALSC_NT) {
        const int l = o / Qj, s = o - l * Qj;
        cplx acc = cmk(0.0, 0.0);
        for (int c = 0; c < R; ++c) acc = cfma(ld(had, (size_t)l * R + c), ld(Vj, (size_t)s * R + c), acc);
        st(rhs, (size_t)l * a.qmax + s, acc);
      }
      __syncthreads();
      // in-place Gauss-Jordan inverse of the Hermitian positive definite normal matrix
      // (no pivoting needed); the reference solves the same system by LU (cp.py:175)
      for (int k = 0; k < r; ++k) {
        if (tid < r) {
          st(rowk, tid, ld(Ai, (size_t)k * r + tid));
          st(colk, tid, ld(Ai, (size_t)tid * r + k));
        }
        __syncthreads();
        const cplx piv = ld(rowk, k);
        if (tid == 0 && !(isfinite(piv.x) && isfinite(piv.y))) status |= 1;
        // zero pivot = zero row/column of the PSD matrix: min-norm (lstsq, cp.py:176-177) solution
        const cplx p = (piv.x == 0.0 && piv.y == 0.0) ? cmk(0.0, 0.0) : crcp(piv);
        for (int e = tid; e < rr; e += ALSC_NT) {
          const int i = e / r, c = e - i * r;
          cplx v;
          if (i == k && c == k) {
            v = p;
          } else if (i == k) {
            v = cmul(ld(rowk, c), p);
          } else if (c == k) {
            v = cmul(cmk(-ld(colk, i).x, -ld(colk, i).y), p);
          } else {
            v = csub(ld(Ai, e), cmul(ld(colk, i), cmul(ld(rowk, c), p)));
          }
          st(Ai, e, v);
        }
        __syncthreads();
      }
      // U_j[s][l] = (A^-1 rhs)[l][s]  (guess.factors[j] = solve(...).T, cp.py:317)
      double* Uj = Us + 2 * (size_t)a.qo[j] * r;
      int nf = 0;
      for (int o = tid; o < Qj * r; o += ALSC_NT) {
        const int s = o / r, l = o - s * r;
        cplx acc = cmk(0.0, 0.0);
        for (int m = 0; m < r; ++m) acc = cfma(ld(Ai, (size_t)l * r + m), ld(rhs, (size_t)m * a.qmax + s), acc);
        if (!(isfinite(acc.x) && isfinite(acc.y))) nf = 1;
        st(Uj, o, acc);
      }
      if (nf) atomicOr(a.info, 2);
      __syncthreads();
      refresh(j);
      __syncthreads();
    }
    done = sweep + 1;
    if (a.need_resid) {   // ||V||^2 - 2 Re sum prod C + Re sum prod G  (cp.py:321-326)
      double ov = 0.0, self = 0.0;
      for (int e = tid; e < r * R; e += ALSC_NT) {
        cplx v = cmk(1.0, 0.0);
        for (int k = 0; k < d; ++k) v = cmul(v, ld(Cs, (size_t)k * r * R + e));
        ov += v.x;
      }
      for (int e = tid; e < rr; e += ALSC_NT) {
        cplx v = cmk(1.0, 0.0);
        for (int k = 0; k < d; ++k) v = cmul(v, ld(Gs, (size_t)k * rr + e));
        self += v.x;
      }
      ov = blk_sum_c(ov, red);
      self = blk_sum_c(self, red2);
      const double resid = sqrt(fmax(norm_sq - 2.0 * ov + self, 0.0));
      if (tid == 0 && a.trace) a.trace[sweep] = resid;
      if (resid <= a.tol * t_norm) break;
      if (prev - resid < a.stall * fmax(t_norm, 1.0)) break;
      prev = resid;
    }
  }
  for (size_t e = tid; e < 2 * (size_t)a.sumq * r; e += ALSC_NT) a.U[e] = Us[e];
  if (status && tid == 0) atomicOr(a.info, 1);
  if (tid == 0) a.info[1] = done;
}

static int als_c_plan(int d, const int* q, int R, int r, AlsCArgs& a, size_t& smem) {
  if (d < 1 || d > TP_MAXD || R < 1 || r < 1 || r > 64 || !q) return TP_EINVAL;
  memset(&a, 0, sizeof(a));
  int sumq = 0, qmax = 0;
  for (int k = 0; k < d; ++k) {
    if (q[k] < 1) return TP_EINVAL;
    a.q[k] = q[k]; a.qo[k] = sumq; sumq += q[k]; qmax = q[k] > qmax ? q[k] : qmax;
  }
  a.d = d; a.R = R; a.r = r; a.sumq = sumq; a.qmax = qmax;
  smem = als_c_smem_doubles(d, sumq, qmax, R, r) * sizeof(double);
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  else cudaGetLastError();
  if (optin <= 0) optin = 227 * 1024;
  if (smem > (size_t)optin) return TP_EUNSUPPORTED;
  return TP_OK;
}

}  // namespace tp

using namespace tp;

extern "C" {

int tp_cp_apply_c128(int d, const int* q, int r_in, const double* F, int n_terms, const double* weights,
                     double scale_re, double scale_im, const int* mat_idx, const double* mats,
                     const long long* mat_off, int n_mats, double* out, int R_out, int col_off, void* stream) {
  if (d < 1 || d > TP_MAXD || r_in < 1 || n_terms < 1 || !F || !out || !q || !weights) return TP_EINVAL;
  if (col_off < 0 || col_off + (long long)n_terms * r_in > R_out) return TP_EINVAL;
  if (n_terms > APC_MAXT) {   // consecutive launches of at most APC_MAXT terms (weights are re/im pairs)
    for (int t0 = 0; t0 < n_terms; t0 += APC_MAXT) {
      const int nt = n_terms - t0 < APC_MAXT ? n_terms - t0 : APC_MAXT;
      const int st = tp_cp_apply_c128(d, q, r_in, F, nt, weights + 2 * (size_t)t0, scale_re, scale_im,
                                      mat_idx ? mat_idx + (size_t)t0 * d : nullptr, mats, mat_off, n_mats, out, R_out,
                                      col_off + t0 * r_in, stream);
      if (st != TP_OK) return st;
    }
    return TP_OK;
  }
  ApplyCArgs a;
  memset(&a, 0, sizeof(a));
  a.d = d; a.r_in = r_in; a.R_out = R_out; a.col_off = col_off; a.n_terms = n_terms;
  long long of = 0, oo = 0;
  int qmax = 1;
  for (int k = 0; k < d; ++k) {
    if (q[k] < 1) return TP_EINVAL;
    a.q[k] = q[k]; a.offF[k] = of; a.offO[k] = oo;
    of += (long long)q[k] * r_in; oo += (long long)q[k] * R_out;
    qmax = q[k] > qmax ? q[k] : qmax;
  }
  a.F = F; a.out = out; a.mats = mats;
  for (int t = 0; t < n_terms; ++t) {
    const double wr = weights[2 * t], wi = weights[2 * t + 1];
    a.w0[2 * t] = scale_re * wr - scale_im * wi;
    a.w0[2 * t + 1] = scale_re * wi + scale_im * wr;
    for (int k = 0; k < d; ++k) {
      const int idx = mat_idx ? mat_idx[t * d + k] : -1;
      if (idx >= n_mats) return TP_EINVAL;
      if (idx >= 0 && (!mats || !mat_off)) return TP_EINVAL;
      a.moff[t][k] = idx < 0 ? -1 : mat_off[idx];
    }
  }
  int zb = (qmax * r_in + 255) / 256;
  zb = zb < 1 ? 1 : (zb > 64 ? 64 : zb);
  cp_apply_c_kernel<<<dim3(n_terms, d, zb), 256, 0, (cudaStream_t)stream>>>(a);
  return cuda_status(cudaGetLastError());
}

size_t tp_cp_inner_c128_ws_bytes(int d, const int* q, int ra, int rb) {
  (void)d; (void)q;
  if (ra < 1 || rb < 1) return 0;
  return align_up(sizeof(double) * 2 * (size_t)ra * rb);
}

int tp_cp_inner_c128(int d, const int* q, int ra, const double* A, int rb, const double* B, double* out, void* ws,
                     size_t ws_bytes, void* stream) {
  if (d < 1 || d > TP_MAXD || ra < 1 || rb < 1 || !A || !B || !out || !q) return TP_EINVAL;
  if (!ws || ws_bytes < tp_cp_inner_c128_ws_bytes(d, q, ra, rb)) return TP_EWORKSPACE;
  for (int k = 0; k < d; ++k) if (q[k] < 1) return TP_EINVAL;
  return launch_inner_c(d, q, ra, A, rb, B, out, static_cast<double*>(ws), (cudaStream_t)stream);
}

size_t tp_cp_als_c128_ws_bytes(int d, const int* q, int R, int r) {
  AlsCArgs a;
  size_t smem = 0;
  if (als_c_plan(d, q, R, r, a, smem) != TP_OK) return 0;
  return align_up(sizeof(double) * 2) + tp_cp_inner_c128_ws_bytes(d, q, R, R);
}

int tp_cp_als_c128(int d, const int* q, int R, const double* V, int r, double* U, int sweeps, double reg, int reg_mode,
                   double tol, double stall, double* trace, int* info, void* ws, size_t ws_bytes, void* stream) {
  if (!V || !U || !info || sweeps < 0 || !(reg >= 0.0)) return TP_EINVAL;
  AlsCArgs a;
  size_t smem = 0;
  int st0 = als_c_plan(d, q, R, r, a, smem);
  if (st0 != TP_OK) return st0;
  if (!ws || ws_bytes < tp_cp_als_c128_ws_bytes(d, q, R, r)) return TP_EWORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  double* nsq = cv.take<double>(2);
  double* part = cv.take<double>(2 * (size_t)R * R);
  a.V = V; a.U = U; a.trace = trace; a.info = info; a.norm_sq = nsq;
  a.sweeps = sweeps; a.reg = reg; a.reg_mode = reg_mode; a.tol = tol; a.stall = stall;
  a.need_resid = (trace != nullptr) || (tol > 0.0) || (stall > -INFINITY);
  cudaError_t e = cudaMemsetAsync(info, 0, 2 * sizeof(int), s);
  if (e != cudaSuccess) return cuda_status(e);
  if (a.need_resid) {
    const int st1 = launch_inner_c(d, q, R, V, R, V, nsq, part, s);   // ||V||^2 (cp.py:186-188)
    if (st1 != TP_OK) return st1;
  }
  e = cudaFuncSetAttribute(als_c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e);
  als_c_kernel<<<1, ALSC_NT, smem, s>>>(a);
  return cuda_status(cudaGetLastError());
}

}  // extern "C"
