// CP-ALS for any output rank r <= ALSG_RMAX and any input rank R: the size-unbounded
// variant behind tp_cp_als_f64 (cp.cp_approx_als, cp.py:266-334) for the problems the
// fused persistent kernels (tp_als.cu) cannot hold -- r > 32, or a target whose
// R-slabs exceed the GPU's aggregate shared memory.  The target streams from HBM /
// L2 every mode update.  Per mode update j (cp.py:310-320), all stream-ordered:
//   had  = prod_{k!=j} C_k                      (r x R, elementwise)
//   rhs  = had V_j^T                            (r x Q_j, DMMA GEMM, cp.py:197-203)
//   A    = prod_{k!=j} G_k + lambda I, A^-1     (one CTA: Cholesky, L^-1, L^-T L^-1;
//                                                cp.py:169-180; a zero pivot of the PSD
//                                                matrix = a zero row -> min-norm, like the
//                                                reference's lstsq fallback)
//   U_j  = (A^-1 rhs)^T                         (DMMA GEMM, cp.py:317)
//   G_j  = U_j^T U_j,  C_j = U_j^T V_j          (DMMA GEMMs, cp.py:318-320)
// After a sweep (only with a trace / stopping rule) the residual by the Gram
// identity (cp.py:321-326) and the tol / stall decisions (cp.py:329-332) are made
// on the device: a stop flag turns every later kernel of the call into a no-op.
#include "tp_common.cuh"
#include "tp_gemm.cuh"
#include <cstring>

namespace tp {

int launch_inner(int d, const int* q, int ra, const double* A, int rb, const double* B, int same,
                 double* out, double* partial, cudaStream_t st);
int inner_tiles(int ra, int rb, int same);

constexpr int ALSG_RMAX = 160;   // A and L^-1 of the r x r normal equations in one CTA's shared memory
constexpr int ALSG_NT = 512;

struct GenState {
  double prev, resid;
  int stop, sweeps;
};

// had[l][c] = prod_{k!=j} C[k][l][c]
__global__ void gen_had_kernel(int d, int j, long long rR, const double* C, double* had, const GenState* gs) {
  if (gs->stop) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rR; e += (long long)gridDim.x * blockDim.x) {
    double v = 1.0;
    for (int k = 0; k < d; ++k)
      if (k != j) v *= C[(size_t)k * rR + e];
    had[e] = v;
  }
}

// A = prod_{k!=j} G_k + lambda I, then Ainv = A^-1 through the Cholesky factor
// (in place in shared memory).  One CTA.
__global__ void __launch_bounds__(ALSG_NT) gen_inverse_kernel(int d, int r, int j, const double* G, double reg,
                                                              int reg_mode, double* Ainv, int* info,
                                                              const GenState* gs) {
  if (gs->stop) return;
  extern __shared__ double sh[];
  const int ld = r + 1, tid = threadIdx.x;
  double* L = sh;                 // [r][ld]
  double* X = L + (size_t)r * ld; // [r][ld]  L^-1
  __shared__ double red[ALSG_NT];
  const size_t rr = (size_t)r * r;
  double dg = 0.0;
  for (int e = tid; e < r * r; e += ALSG_NT) {
    const int i = e / r, c = e - i * r;
    double v = 1.0;
    for (int k = 0; k < d; ++k)
      if (k != j) v *= G[(size_t)k * rr + e];
    L[i * ld + c] = v;
    if (i == c) dg += v;
  }
  double lam = reg;
  if (reg_mode) {   // reference rule lambda = reg * max(tr A, 0) / r (cp.py:171-173), fixed-order sum
    red[tid] = dg;
    __syncthreads();
    for (int w = ALSG_NT / 2; w > 0; w >>= 1) {
      if (tid < w) red[tid] += red[tid + w];
      __syncthreads();
    }
    lam = reg * fmax(red[0], 0.0) / (double)r;
  }
  __syncthreads();
  for (int i = tid; i < r; i += ALSG_NT) L[i * ld + i] += lam;
  __syncthreads();
  // right-looking Cholesky, lower triangle
  int bad = 0;
  for (int p = 0; p < r; ++p) {
    const double dpp = L[p * ld + p];
    if (dpp < 0.0 || !isfinite(dpp)) bad = 1;
    const bool zero = !(dpp > 0.0);   // zero row of the PSD matrix: min-norm (lstsq, cp.py:176-177)
    const double dsq = zero ? 0.0 : sqrt(dpp), inv = zero ? 0.0 : 1.0 / dsq;
    __syncthreads();
    if (tid == 0) L[p * ld + p] = dsq;
    for (int i = p + 1 + tid; i < r; i += ALSG_NT) L[i * ld + p] *= inv;
    __syncthreads();
    const int m = r - p - 1;
    for (int e = tid; e < m * m; e += ALSG_NT) {
      const int i = p + 1 + e / m, c = p + 1 + e % m;
      if (c <= i) L[i * ld + c] = fma(-L[i * ld + p], L[c * ld + p], L[i * ld + c]);
    }
    __syncthreads();
  }
  if (bad && tid == 0) atomicOr(info, 1);
  // X = L^-1, column-parallel forward substitution (zero diagonal -> zero row/column)
  for (int c = tid; c < r; c += ALSG_NT) {
    for (int i = 0; i < r; ++i) {
      if (i < c) { X[i * ld + c] = 0.0; continue; }
      double acc = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) acc = fma(-L[i * ld + k], X[k * ld + c], acc);
      const double lii = L[i * ld + i];
      X[i * ld + c] = lii > 0.0 ? acc / lii : 0.0;
    }
  }
  __syncthreads();
  // Ainv = X^T X (symmetric)
  for (int e = tid; e < r * r; e += ALSG_NT) {
    const int i = e / r, c = e - i * r;
    const int k0 = i > c ? i : c;
    double acc = 0.0;
    for (int k = k0; k < r; ++k) acc = fma(X[k * ld + i], X[k * ld + c], acc);
    Ainv[e] = acc;
  }
}

// flag non-finite coefficients of the new U_j (cp.py:178-179)
__global__ void gen_check_kernel(long long n, const double* u, int* info, const GenState* gs) {
  if (gs->stop) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    if (!isfinite(u[e])) { atomicOr(info, 2); return; }
}

// residual after a sweep (cp.py:321-332): ||V||^2 - 2 sum prod C + sum prod G, trace,
// tol / stall decisions.  One CTA, fixed-order reductions.
__global__ void __launch_bounds__(ALSG_NT) gen_resid_kernel(int d, int r, long long R, const double* C, const double* G,
                                                            const double* nsq, double tol, double stall, int sweep,
                                                            double* trace, GenState* gs, int* info) {
  if (gs->stop) return;
  __shared__ double red[ALSG_NT];
  const int tid = threadIdx.x;
  const long long rR = (long long)r * R, rr = (long long)r * r;
  double ov = 0.0, self = 0.0;
  for (long long e = tid; e < rR; e += ALSG_NT) {
    double v = 1.0;
    for (int k = 0; k < d; ++k) v *= C[(size_t)k * rR + e];
    ov += v;
  }
  for (long long e = tid; e < rr; e += ALSG_NT) {
    double v = 1.0;
    for (int k = 0; k < d; ++k) v *= G[(size_t)k * rr + e];
    self += v;
  }
  red[tid] = self - 2.0 * ov;
  __syncthreads();
  for (int w = ALSG_NT / 2; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  if (tid == 0) {
    const double ns = fmax(*nsq, 0.0), tn = sqrt(ns);
    const double resid = sqrt(fmax(ns + red[0], 0.0));
    if (trace) trace[sweep] = resid;
    gs->sweeps = sweep + 1;
    info[1] = sweep + 1;
    if (resid <= tol * tn) gs->stop = 1;
    else if (gs->prev - resid < stall * fmax(tn, 1.0)) gs->stop = 1;
    gs->prev = resid;
  }
}

__global__ void gen_init_state(GenState* gs, int* info, int sweeps, int need_resid) {
  gs->prev = INFINITY;
  gs->resid = 0.0;
  gs->stop = 0;
  gs->sweeps = 0;
  info[0] = 0;
  info[1] = need_resid ? 0 : sweeps;
}

struct GenLayout {
  size_t C, G, had, rhs, Ainv, nsq, state, part, inner, total;
};

static GenLayout gen_layout(int d, const int* q, int R, int r) {
  GenLayout L{};
  int qmax = 0;
  for (int k = 0; k < d; ++k) qmax = q[k] > qmax ? q[k] : qmax;
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t at = o; o += align_up(bytes); return at; };
  L.C = take(8 * (size_t)d * r * R);
  L.G = take(8 * (size_t)d * r * r);
  L.had = take(8 * (size_t)r * R);
  L.rhs = take(8 * (size_t)r * qmax);
  L.Ainv = take(8 * (size_t)r * r);
  L.nsq = take(8);
  L.state = take(sizeof(GenState));
  L.part = take(8 * 16 * (size_t)r * (r > qmax ? r : qmax));   // split-K partials of the K = R / K = Q GEMMs
  L.inner = take(8 * (size_t)inner_tiles(R, R, 1));
  L.total = o;
  return L;
}

int als_generic_supported(int d, const int* q, int R, int r) {
  if (d < 1 || d > TP_MAXD_GEN || R < 1 || r < 1 || r > ALSG_RMAX || !q) return 0;
  for (int k = 0; k < d; ++k) if (q[k] < 1) return 0;
  return 1;
}

size_t als_generic_ws_bytes(int d, const int* q, int R, int r) {
  if (!als_generic_supported(d, q, R, r)) return 0;
  return gen_layout(d, q, R, r).total;
}

static cudaError_t gemm_split(BGemm g, double* part, size_t part_doubles, const GenState* gs, cudaStream_t st) {
  g.skip = &gs->stop;
  const int ks = bgemm_pick_split(g, 148, 4);
  if (ks > 1 && (size_t)g.M * g.N * ks <= part_doubles) { g.ksplit = ks; g.part = part; }
  return bgemm_launch(g, st);
}

int als_generic_run(int d, const int* q, int R, const double* V, int r, double* U, int sweeps, double reg,
                    int reg_mode, double tol, double stall, double* trace, int* info, void* ws, size_t ws_bytes,
                    cudaStream_t st) {
  if (!als_generic_supported(d, q, R, r)) return TP_EUNSUPPORTED;
  const GenLayout Lo = gen_layout(d, q, R, r);
  if (!ws || ws_bytes < Lo.total) return TP_EWORKSPACE;
  char* base = static_cast<char*>(ws);
  double* C = reinterpret_cast<double*>(base + Lo.C);
  double* G = reinterpret_cast<double*>(base + Lo.G);
  double* had = reinterpret_cast<double*>(base + Lo.had);
  double* rhs = reinterpret_cast<double*>(base + Lo.rhs);
  double* Ainv = reinterpret_cast<double*>(base + Lo.Ainv);
  double* nsq = reinterpret_cast<double*>(base + Lo.nsq);
  GenState* gs = reinterpret_cast<GenState*>(base + Lo.state);
  double* part = reinterpret_cast<double*>(base + Lo.part);
  double* inner = reinterpret_cast<double*>(base + Lo.inner);
  int qmax = 0;
  for (int k = 0; k < d; ++k) qmax = q[k] > qmax ? q[k] : qmax;
  const size_t part_doubles = 16 * (size_t)r * (r > qmax ? r : qmax);
  long long offV[TP_MAXD_GEN], offU[TP_MAXD_GEN];
  long long ov = 0, ou = 0;
  for (int k = 0; k < d; ++k) { offV[k] = ov; offU[k] = ou; ov += (long long)q[k] * R; ou += (long long)q[k] * r; }
  const bool need_resid = trace || tol > 0.0 || stall > -INFINITY;
  gen_init_state<<<1, 1, 0, st>>>(gs, info, sweeps, need_resid ? 1 : 0);
  if (need_resid) {
    const int s = launch_inner(d, q, R, V, R, V, 1, nsq, inner, st);   // ||V||^2 (cp.py:186-188)
    if (s != TP_OK) return s;
  }
  cudaError_t e = cudaGetLastError();
  // set-up: C_k = U_k^T V_k, G_k = U_k^T U_k  (cp.py:305-307)
  for (int k = 0; k < d && e == cudaSuccess; ++k) {
    e = gemm_split(bgemm_desc(r, R, q[k], U + offU[k], 1, r, V + offV[k], R, 1, C + (size_t)k * r * R, R, 1), part,
                   part_doubles, gs, st);
    if (e == cudaSuccess)
      e = gemm_split(bgemm_desc(r, r, q[k], U + offU[k], 1, r, U + offU[k], r, 1, G + (size_t)k * r * r, r, 1), part,
                     part_doubles, gs, st);
  }
  const size_t ism = sizeof(double) * 2 * (size_t)r * (r + 1);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(gen_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ism);
  const long long rR = (long long)r * R;
  const int hb = (int)((rR + 255) / 256 < 1184 ? (rR + 255) / 256 : 1184);
  for (int sweep = 0; sweep < sweeps && e == cudaSuccess; ++sweep) {
    for (int j = 0; j < d && e == cudaSuccess; ++j) {
      const int Qj = q[j];
      gen_had_kernel<<<hb, 256, 0, st>>>(d, j, rR, C, had, gs);
      // rhs[l][s] = sum_c had[l][c] V_j[s][c]
      e = gemm_split(bgemm_desc(r, Qj, R, had, R, 1, V + offV[j], 1, R, rhs, Qj, 1), part, part_doubles, gs, st);
      if (e != cudaSuccess) break;
      gen_inverse_kernel<<<1, ALSG_NT, ism, st>>>(d, r, j, G, reg, reg_mode, Ainv, info, gs);
      // U_j[s][i] = sum_m rhs[m][s] Ainv[m][i]   (Ainv symmetric)
      e = gemm_split(bgemm_desc(Qj, r, r, rhs, 1, Qj, Ainv, r, 1, U + offU[j], r, 1), part, part_doubles, gs, st);
      if (e != cudaSuccess) break;
      gen_check_kernel<<<(int)(((long long)Qj * r + 255) / 256), 256, 0, st>>>((long long)Qj * r, U + offU[j], info, gs);
      e = gemm_split(bgemm_desc(r, r, Qj, U + offU[j], 1, r, U + offU[j], r, 1, G + (size_t)j * r * r, r, 1), part,
                     part_doubles, gs, st);
      if (e == cudaSuccess)
        e = gemm_split(bgemm_desc(r, R, Qj, U + offU[j], 1, r, V + offV[j], R, 1, C + (size_t)j * r * R, R, 1), part,
                       part_doubles, gs, st);
      if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (need_resid && e == cudaSuccess) {
      gen_resid_kernel<<<1, ALSG_NT, 0, st>>>(d, r, R, C, G, nsq, tol, stall, sweep, trace, gs, info);
      e = cudaGetLastError();
    }
  }
  return cuda_status(e);
}

}  // namespace tp
