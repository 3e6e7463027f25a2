// CP inner products (K3 target Gram norm, cp.inner_product) and separable
// operator apply (K1, operators.apply) for sm_100a.
#include "tp_common.cuh"
#include <cstdio>
#include <cstring>

namespace tp {

static thread_local char g_last_error[256] = "";

void set_last_error(cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s", cudaGetErrorString(e));
}

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return TP_OK;
  set_last_error(e);
  return TP_ECUDA;
}

// ---------------------------------------------------------------------------
// K3: <A, B> = sum_{l,m} prod_k (A_k^T B_k)[l, m]   (cp.py:111-121)
//
// One CTA per 32x32 tile of the (l, m) term-pair plane; 4 warps, each owning
// a 16x16 sub-tile as 2x2 DMMA m8n8k4 accumulators.  For every mode the
// per-mode Gram tile is accumulated over Q in 32-row chunks staged in shared
// memory, then folded into the running Hadamard product held in registers;
// the d Gram matrices are never materialised.  Symmetric calls (A == B) only
// visit upper tiles and double the off-diagonal ones.
// ---------------------------------------------------------------------------
constexpr int IP_T = 32;      // tile edge
constexpr int IP_KC = 32;     // Q rows per staged chunk
constexpr int IP_LD = 36;     // padded smem row (conflict-free fragment loads)

struct InnerArgs {
  int d, ra, rb, same, ntl, ntm;
  int q[TP_MAXD_GEN];
  long long offA[TP_MAXD_GEN], offB[TP_MAXD_GEN];
  const double* A;
  const double* B;
  double* partial;
};

__global__ void __launch_bounds__(128) cp_inner_tiles(InnerArgs a) {
  __shared__ double sA[IP_KC][IP_LD];
  __shared__ double sB[IP_KC][IP_LD];
  __shared__ double wsum[4];
  int tl, tm;
  if (a.same) {
    // enumerate upper tiles (tl <= tm) row by row
    int t = blockIdx.x, row = 0, len = a.ntl;
    while (t >= len) { t -= len; ++row; --len; }
    tl = row; tm = row + t;
  } else {
    tl = blockIdx.x / a.ntm; tm = blockIdx.x % a.ntm;
  }
  const int l0 = tl * IP_T, m0 = tm * IP_T;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wl = (warp >> 1) * 16, wm = (warp & 1) * 16;
  double prod[2][2][2];
  for (int k = 0; k < a.d; ++k) {
    double acc[2][2][2] = {};
    const int Q = a.q[k];
    const double* Ak = a.A + a.offA[k];
    const double* Bk = a.B + a.offB[k];
    for (int s0 = 0; s0 < Q; s0 += IP_KC) {
      __syncthreads();
      for (int e = tid; e < IP_KC * IP_T; e += 128) {
        int rs = e / IP_T, c = e % IP_T;
        int s = s0 + rs;
        sA[rs][c] = (s < Q && l0 + c < a.ra) ? Ak[(long long)s * a.ra + l0 + c] : 0.0;
        sB[rs][c] = (s < Q && m0 + c < a.rb) ? Bk[(long long)s * a.rb + m0 + c] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < IP_KC; kk += 4) {
        const int rr = kk + (lane & 3), cc = lane >> 2;
        double fa0 = sA[rr][wl + cc], fa1 = sA[rr][wl + 8 + cc];
        double fb0 = sB[rr][wm + cc], fb1 = sB[rr][wm + 8 + cc];
        dmma_8x8x4(acc[0][0][0], acc[0][0][1], fa0, fb0);
        dmma_8x8x4(acc[0][1][0], acc[0][1][1], fa0, fb1);
        dmma_8x8x4(acc[1][0][0], acc[1][0][1], fa1, fb0);
        dmma_8x8x4(acc[1][1][0], acc[1][1][1], fa1, fb1);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) prod[i][j][h] = (k == 0) ? acc[i][j][h] : prod[i][j][h] * acc[i][j][h];
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) s += prod[i][j][0] + prod[i][j][1];
  s = warp_sum(s);
  if (lane == 0) wsum[warp] = s;
  __syncthreads();
  if (tid == 0) {
    double t = ((wsum[0] + wsum[1]) + wsum[2]) + wsum[3];
    if (a.same && tl != tm) t *= 2.0;
    a.partial[blockIdx.x] = t;
  }
}

// deterministic fixed-order sum of n partials into *out
__global__ void __launch_bounds__(256) sum_partials(const double* __restrict__ part, int n, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

int inner_tiles(int ra, int rb, int same) {
  int ntl = (ra + IP_T - 1) / IP_T, ntm = (rb + IP_T - 1) / IP_T;
  return same ? ntl * (ntl + 1) / 2 : ntl * ntm;
}

int launch_inner(int d, const int* q, int ra, const double* A, int rb, const double* B, int same,
                 double* out, double* partial, cudaStream_t st) {
  InnerArgs a;
  memset(&a, 0, sizeof(a));
  a.d = d; a.ra = ra; a.rb = rb; a.same = same;
  a.ntl = (ra + IP_T - 1) / IP_T; a.ntm = (rb + IP_T - 1) / IP_T;
  long long oa = 0, ob = 0;
  for (int k = 0; k < d; ++k) {
    a.q[k] = q[k]; a.offA[k] = oa; a.offB[k] = ob;
    oa += (long long)q[k] * ra; ob += (long long)q[k] * rb;
  }
  a.A = A; a.B = B; a.partial = partial;
  int nt = inner_tiles(ra, rb, same);
  cp_inner_tiles<<<nt, 128, 0, st>>>(a);
  sum_partials<<<1, 256, 0, st>>>(partial, nt, out);
  return cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// K1: separable operator apply into a concatenated target (operators.py:48-62)
// grid: (term, mode, row-block); each thread produces output entries
// out_k[s, col_off + t*r_in + c] for a (s, c) range.
// ---------------------------------------------------------------------------
constexpr int AP_MAXT = 64;

struct ApplyArgs {
  int d, r_in, R_out, col_off, n_terms;
  int q[TP_MAXD_GEN];
  long long offF[TP_MAXD_GEN], offO[TP_MAXD_GEN];
  const double* F;
  double* out;
  const double* mats;
  double w0[AP_MAXT];                 // scale * weight per term (mode 0 only)
  long long moff[AP_MAXT][TP_MAXD_GEN];   // matrix element offset, -1 = identity
};

// the argument block (~5 KB) is passed by value (CUDA >= 12.1 allows 32 KB of
// kernel parameters), so the launch is capturable in a CUDA graph.
__global__ void __launch_bounds__(256) cp_apply_kernel(const __grid_constant__ ApplyArgs a) {
  extern __shared__ double aps[];
  const int t = blockIdx.x, k = blockIdx.y;
  const int Q = a.q[k], r = a.r_in;
  const double* Fk = a.F + a.offF[k];
  double* Ok = a.out + a.offO[k];
  const long long mo = a.moff[t][k];
  const double sc = (k == 0) ? a.w0[t] : 1.0;
  const int col = a.col_off + t * r;
  // this CTA's rows [s0, s1) of the (term, mode) block
  const int s0 = (int)((long long)Q * blockIdx.z / gridDim.z), s1 = (int)((long long)Q * (blockIdx.z + 1) / gridDim.z);
  const int nr = s1 - s0;
  if (mo >= 0 && (size_t)(nr * Q + Q * r) * sizeof(double) <= 48 * 1024) {
    // operator rows and the factor staged in shared memory (coalesced), then the same
    // sequential-fma matvec as the direct path (bitwise identical)
    double* Es = aps;              // [nr][Q]
    double* Fs = aps + nr * Q;     // [Q][r]
    const double* E = a.mats + mo + (long long)s0 * Q;
    for (int e = threadIdx.x; e < nr * Q; e += 256) Es[e] = __ldg(E + e);
    for (int e = threadIdx.x; e < Q * r; e += 256) Fs[e] = __ldg(Fk + e);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * r; e += 256) {
      const int sl = e / r, c = e - sl * r;
      const double* er = Es + sl * Q;
      double acc = 0.0;
#pragma unroll 4
      for (int u = 0; u < Q; ++u) acc = fma(er[u], Fs[u * r + c], acc);
      Ok[(long long)(s0 + sl) * a.R_out + col + c] = sc * acc;
    }
    return;
  }
  for (int e = threadIdx.x; e < nr * r; e += blockDim.x) {
    const int s = s0 + e / r, c = e % r;
    double v;
    if (mo < 0) {
      v = Fk[(long long)s * r + c];
    } else {
      const double* E = a.mats + mo + (long long)s * Q;
      double acc = 0.0;
      for (int u = 0; u < Q; ++u) acc = fma(__ldg(E + u), __ldg(Fk + (long long)u * r + c), acc);
      v = acc;
    }
    Ok[(long long)s * a.R_out + col + c] = sc * v;
  }
}

}  // namespace tp

using namespace tp;

// Weight contractions of a CP tensor (moments, point evaluation):
//   out[w] = sum_l prod_k ( W[w][k] . F_k[:, l] )
// (cp.py:84-95 evaluate with basis values as W; diagnostics.py:60-64 _contract with
// integration weights).  One CTA per weight set, terms over the threads, W staged
// in shared memory, fixed-order block reduction.
constexpr int CT_NT = 256;

struct QOff { int v[TP_MAXD_GEN + 1]; };

__global__ void __launch_bounds__(CT_NT) cp_contract_kernel(int d, const __grid_constant__ QOff qo_, int sumq, int R,
                                                            const double* __restrict__ F,
                                                            const double* __restrict__ W, double* out) {
  extern __shared__ double ws_[];
  double* w = ws_;                 // [sumq]
  double* red = ws_ + sumq;        // [CT_NT]
  const int* qo = qo_.v;
  const int wi = blockIdx.x, tid = threadIdx.x;
  for (int e = tid; e < sumq; e += CT_NT) w[e] = W[(size_t)wi * sumq + e];
  __syncthreads();
  double acc = 0.0;
  for (int l = tid; l < R; l += CT_NT) {
    double prod = 1.0;
    for (int k = 0; k < d; ++k) {
      const int q0 = qo[k], Q = qo[k + 1] - q0;
      const double* Fk = F + (size_t)q0 * R + l;   // mode k block is (Q_k, R) row-major at R * q0
      double dot = 0.0;
      for (int s = 0; s < Q; ++s) dot = fma(w[q0 + s], Fk[(size_t)s * R], dot);
      prod *= dot;
    }
    acc += prod;
  }
  red[tid] = acc;
  __syncthreads();
  for (int h = CT_NT / 2; h > 0; h >>= 1) {
    if (tid < h) red[tid] += red[tid + h];
    __syncthreads();
  }
  if (tid == 0) out[wi] = red[0];
}

extern "C" {

const char* tp_version(void) { return "tpde_b200 0.1.0 (sm_100a)"; }

const char* tp_status_string(int s) {
  switch (s) {
    case TP_OK: return "ok";
    case TP_EINVAL: return "invalid argument";
    case TP_ENONFINITE: return "non-finite coefficients";
    case TP_ENOTPD: return "normal equations not positive definite";
    case TP_ECUDA: return "CUDA error";
    case TP_EWORKSPACE: return "workspace too small";
    case TP_EUNSUPPORTED: return "unsupported size";
    default: return "unknown status";
  }
}

const char* tp_last_error(void) { return g_last_error; }

int tp_device_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n;
}

size_t tp_cp_inner_ws_bytes(int d, const int* q, int ra, int rb) {
  (void)d; (void)q;
  return align_up(sizeof(double) * (size_t)inner_tiles(ra, rb, 0));
}

int tp_cp_inner_f64(int d, const int* q, int ra, const double* A, int rb, const double* B,
                    int same, double* out, void* ws, size_t ws_bytes, void* stream) {
  if (d < 1 || d > TP_MAXD_GEN || ra < 1 || rb < 1 || !A || !B || !out || !q) return TP_EINVAL;
  for (int k = 0; k < d; ++k) if (q[k] < 1) return TP_EINVAL;
  if (same && (ra != rb || A != B)) return TP_EINVAL;
  if (ws_bytes < sizeof(double) * (size_t)inner_tiles(ra, rb, same)) return TP_EWORKSPACE;
  return launch_inner(d, q, ra, A, rb, B, same, out, static_cast<double*>(ws), (cudaStream_t)stream);
}

int tp_cp_apply_f64(int d, const int* q, int r_in, const double* F, int n_terms,
                    const double* weights, double scale, const int* mat_idx,
                    const double* mats, const long long* mat_off, int n_mats,
                    double* out, int R_out, int col_off, void* stream) {
  if (d < 1 || d > TP_MAXD_GEN || r_in < 1 || n_terms < 1 || !F || !out || !q || !weights) return TP_EINVAL;
  if (col_off < 0 || col_off + (long long)n_terms * r_in > R_out) return TP_EINVAL;
  if (n_terms > AP_MAXT) {   // more terms than one argument block holds: consecutive launches
    for (int t0 = 0; t0 < n_terms; t0 += AP_MAXT) {
      const int nt = n_terms - t0 < AP_MAXT ? n_terms - t0 : AP_MAXT;
      const int st = tp_cp_apply_f64(d, q, r_in, F, nt, weights + t0, scale, mat_idx ? mat_idx + (size_t)t0 * d : nullptr,
                                     mats, mat_off, n_mats, out, R_out, col_off + t0 * r_in, stream);
      if (st != TP_OK) return st;
    }
    return TP_OK;
  }
  ApplyArgs a;
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
    a.w0[t] = scale * weights[t];
    for (int k = 0; k < d; ++k) {
      int idx = mat_idx ? mat_idx[t * d + k] : -1;
      if (idx >= n_mats) return TP_EINVAL;
      if (idx >= 0 && (!mats || !mat_off)) return TP_EINVAL;
      a.moff[t][k] = idx < 0 ? -1 : mat_off[idx];
    }
  }
  cudaStream_t st = (cudaStream_t)stream;
  int zb = (qmax * r_in + 255) / 256;
  zb = zb < 1 ? 1 : (zb > 64 ? 64 : zb);
  if (zb > qmax) zb = qmax;
  dim3 grid(n_terms, d, zb);
  cp_apply_kernel<<<grid, 256, 48 * 1024, st>>>(a);
  return cuda_status(cudaGetLastError());
}


int tp_cp_contract_f64(int d, const int* q, int R, const double* F, int nw, const double* W, double* out,
                       void* stream) {
  if (d < 1 || d > TP_MAXD_GEN || R < 1 || nw < 0 || !q || !F || !out || (nw > 0 && !W)) return TP_EINVAL;
  QOff qo;
  qo.v[0] = 0;
  for (int k = 0; k < d; ++k) {
    if (q[k] < 1) return TP_EINVAL;
    qo.v[k + 1] = qo.v[k] + q[k];
  }
  if (nw == 0) return TP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = sizeof(double) * ((size_t)qo.v[d] + CT_NT);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(cp_contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e);
  }
  cp_contract_kernel<<<nw, CT_NT, smem, st>>>(d, qo, qo.v[d], R, F, W, out);
  return cuda_status(cudaGetLastError());
}
}  // extern "C"
