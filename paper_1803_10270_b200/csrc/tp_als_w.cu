// Gram-space CP-ALS (cp.cp_approx_als, cp.py:266-334) for large, well-conditioned
// truncations (BASELINE config 1: d=6, Q=256, R=512, r=32): one launch runs every sweep.
//
// The mode update of the reference (cp.py:311-320)
//     had_j = prod_{k != j} C_k,  A_j = prod_{k != j} G_k + lambda I,
//     U_j = V_j had_j^T A_j^-1,   C_j = U_j^T V_j,   G_j = U_j^T U_j
// only ever uses U_j through its cross C_j (r x R) and Gram G_j (r x r).  With the
// target Grams W_j = V_j^T V_j (R x R, one batched GEMM before the sweeps) the same
// update is, in exact arithmetic,
//     T_j = had_j W_j,   C_j = X_j T_j,   G_j = sym(C_j had_j^T X_j),   X_j = A_j^-1,
// i.e. the sweeps never touch the Q dimension: no reduction over the rows of the
// factor, one all-gather of had_j (r x R) per mode update instead of a reduce-scatter
// plus an all-gather, and U_j = V_j had_j^T X_j is formed once after the last sweep.
//
// Grid: P = ceil(R / 8) CTAs; CTA c owns target terms (columns of every C_k) [8c, 8c+8).
// A round (sweep s, mode j), 256 threads:
//   warps 0-3  T_j[:, own] = had_j W_j[:, own]: the K range (all R terms) split over the
//              warps; had_j comes piecewise from the producers' global "pieces", fragments
//              straight from L2 into registers (16-byte loads, double-buffered chunks of
//              four pieces), DMMA; then the matrix Newton-Schulz update of the previous
//              round (X1 = X0 Tn) while they wait at the join;
//   warps 4-7  meanwhile: sum this CTA's share of the partial Grams C had^T X of the
//              previous update over all producers (fixed order) and publish it; gather the
//              sum, G_{j-1} = sym(.), A_j, and the Newton-Schulz residual of the previous
//              sweep's X_j (Tn = 2I - A_j X_j, accepted when |I - A_j X_j| <= 1e-8; else,
//              and in the first sweep, the exact sweep-operator inverse on these warps);
//   all        C_j[:, own] = X_j T_j applied as X0 (Tn T_j), Y = X_j had_j[:, own], the
//              partial Gram C_j[:, own] Y^T and the own columns of had_{j+1}, written as
//              this CTA's piece of the next round.
// Synchronisation is carried by the data: exchange buffers are armed with all-ones words
// (a NaN no arithmetic produces), readers spin on the words they need, writers re-arm
// their words one sweep before the next use -- no flags, no fences, one L2 hop per
// exchange.  Everything every CTA computes redundantly (G, A, X) is bitwise identical
// across CTAs (fixed summation orders), so stopping and fallback decisions are uniform,
// and results are bitwise reproducible.
//
// Accuracy: C_j = X (had W) carries an error ~ eps cond(A_j) relative to the direct
// form; the kernel therefore estimates cond(A_j) from the pivots of every exact inverse
// and, above a.cond_max, writes nothing and raises *redo: the direct cluster-row kernel
// (tp_als_rows.cu), launched behind it, then reruns the truncation (it returns at once
// otherwise).
#include "tp_als_w.cuh"
#include "tp_gemm.cuh"
#include <cfloat>
#include <cmath>
#include <cstring>

namespace tp {

int launch_inner(int d, const int* q, int ra, const double* A, int rb, const double* B, int same,
                 double* out, double* partial, cudaStream_t st);
int inner_tiles(int ra, int rb, int same);

constexpr int WK_NT = 256;
constexpr int WK_RH = 36;                 // row stride of the r x r matrices (== 4 mod 16: conflict-free fragments)
constexpr int WK_MAT = W_RM * WK_RH;

struct WSmem {
  double *Cs, *hads, *Tp, *Ts, *Tl, *Tx, *Gs, *Xs, *Am, *Tn, *X1, *Ms, *Yp, *Ys, *part, *pub, *red;
  uint64_t* bar;   // [2] pair exchange (round parity)
  int* flag;   // [0]: Newton-Schulz accepted, [1]: a poll timed out
};

__host__ __device__ inline size_t wk_smem_doubles(int d) {
  return (size_t)d * W_HAD + 2 * W_HAD + 4 * W_HAD + W_HAD + 2 * (size_t)d * WK_MAT + 5 * (size_t)WK_MAT + 8 * W_HAD +
         8 * WK_RH + 8 + 80 + WK_NT + 8 + 3 * W_HAD + 4;
}

__device__ inline WSmem wk_carve(double* b, int d) {
  WSmem s;
  s.Cs = b; b += (size_t)d * W_HAD;
  s.hads = b; b += 2 * W_HAD;
  s.Tp = b; b += 4 * W_HAD;
  s.Ts = b; b += W_HAD;
  s.Tl = b; b += W_HAD;
  s.Tx = b; b += 2 * W_HAD;
  s.Gs = b; b += (size_t)d * WK_MAT;
  s.Xs = b; b += (size_t)d * WK_MAT;
  s.Am = b; b += WK_MAT;
  s.Tn = b; b += 2 * WK_MAT;   // two buffers (round parity): the previous round's stays readable
  s.X1 = b; b += WK_MAT;
  s.Ms = b; b += WK_MAT;
  s.Yp = b; b += 8 * W_HAD;
  s.Ys = b; b += 8 * WK_RH;
  s.part = b; b += 8;
  s.pub = b; b += 80;
  s.red = b; b += WK_NT;
  s.flag = reinterpret_cast<int*>(b); b += 2;
  s.bar = reinterpret_cast<uint64_t*>(b);
  return s;
}

__device__ __forceinline__ void wk_bar(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// 32 x 32 x 32 product P = A B (row stride WK_RH) on the four warps [w0, w0 + 4): warp w owns the
// 2 x 2 block of 8 x 8 tiles (2 (w / 2) + {0, 1}, 2 (w % 2) + {0, 1}).  mode 0: out = 2I - P and
// returns this thread's max |I - P|_ic over i, c < r; mode 1: out = P.
__device__ double wk_gemm32(const double* A, const double* B, double* out, int r, int mode, int w0) {
  const int warp = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
  const uint32_t a32 = smem_u32(A), b32 = smem_u32(B), o32 = smem_u32(out);
  const int bm = 2 * (warp >> 1), bn = 2 * (warp & 1);
  double acc[2][2][2] = {};
  const uint32_t ar = a32 + 8u * (uint32_t)((bm * 8 + (lane >> 2)) * WK_RH + (lane & 3));
  const uint32_t bc = b32 + 8u * (uint32_t)((lane & 3) * WK_RH + bn * 8 + (lane >> 2));
#pragma unroll
  for (int kk = 0; kk < W_RM / 4; ++kk) {
    double fa[2], fb[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      fa[q] = lds64(ar + 8u * (uint32_t)(q * 8 * WK_RH) + 32u * (uint32_t)kk);
      fb[q] = lds64(bc + 64u * (uint32_t)q + 32u * (uint32_t)(kk * WK_RH));
    }
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int p = 0; p < 2; ++p) dmma_8x8x4(acc[q][p][0], acc[q][p][1], fa[q], fb[p]);
  }
  double emax = 0.0;
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int i = (bm + q) * 8 + (lane >> 2);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = (bn + p) * 8 + 2 * (lane & 3) + h;
        const double dl = (i == c) ? 1.0 : 0.0;
        if (mode == 0) {
          out[i * WK_RH + c] = 2.0 * dl - acc[q][p][h];
          if (i < r && c < r) emax = fmax(emax, fabs(dl - acc[q][p][h]));
        } else {
          out[i * WK_RH + c] = acc[q][p][h];
        }
      }
    }
  (void)o32;
  return emax;
}

// A^-1 (A = sm.Am, symmetric positive definite) -> out by the symmetric sweep operator
// (Gauss-Jordan, one pivot per named barrier) on the 128 threads of warps 4-7 -- the other warps
// keep working on the T product: thread t owns row t / 4, columns t % 4 + 4 u.  *ratio = max
// diagonal / min pivot (a lower bound of cond A; inf when a pivot is <= 0 or not finite);
// identical in every thread and every CTA.
__device__ void wk_inverse(const WSmem& sm, int r, double* out, double* ratio) {
  constexpr int EPT = W_RM / 4;
  const int t = threadIdx.x - 128, i = t >> 2, c0 = t & 3;
  double* pub = sm.pub;
  double v[EPT];
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int c = c0 + 4 * u;
    v[u] = (i < r && c < r) ? sm.Am[i * WK_RH + c] : 0.0;
  }
  double dmax = 0.0, dmin = INFINITY;
  for (int k = 0; k < r; ++k) dmax = fmax(dmax, sm.Am[k * WK_RH + k]);
  if (i == 0)
#pragma unroll
    for (int u = 0; u < EPT; ++u) pub[c0 + 4 * u] = v[u];
  wk_bar(1, 128);
  for (int k = 0; k < r; ++k) {
    const double* rk = pub + (k & 1) * 36;
    double* rn = pub + ((k + 1) & 1) * 36;
    const double d = rk[k];
    dmin = (d > 0.0 && isfinite(d)) ? fmin(dmin, d) : 0.0;
    const double id = (d == 0.0) ? 0.0 : rcp_nr(d);
    const double f = (i < r ? rk[i] : 0.0) * id;
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + 4 * u;
      const double akc = rk[c];
      double nv = fma(-f, akc, v[u]);
      nv = (c == k) ? f : nv;
      nv = (i == k) ? ((c == k) ? -id : akc * id) : nv;
      v[u] = nv;
    }
    if (i == k + 1)
#pragma unroll
      for (int u = 0; u < EPT; ++u) rn[c0 + 4 * u] = v[u];
    wk_bar(1, 128);
  }
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int c = c0 + 4 * u;
    out[i * WK_RH + c] = (i < r && c < r) ? -v[u] : 0.0;
  }
  *ratio = (dmin > 0.0) ? dmax / dmin : INFINITY;
  wk_bar(1, 128);
}

// deterministic block sum (all threads call; result valid in all threads)
__device__ inline double wk_block_sum(double v, double* red) {
  const int tid = threadIdx.x;
  red[tid] = v;
  __syncthreads();
  for (int w = WK_NT / 2; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

// remote store into the peer CTA of the pair, completing bytes on the peer's mbarrier
__device__ __forceinline__ void wk_st_async_v2(uint32_t addr, double x, double y, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
               "d"(x), "d"(y), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void wk_cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// ---- data-carried synchronisation ------------------------------------------------------
// Exchange buffers start as all-ones words (a quiet NaN no arithmetic produces); a reader
// spins on the words it needs until none is the sentinel (relaxed gpu-scope loads from L2:
// no flag, no fence, no second round trip), and the writer re-arms its words of the other
// sweep parity one sweep before their next use.
__device__ __forceinline__ double wk_ldv(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
// (the high word alone identifies the sentinel: no stored double has an all-ones high word)
__device__ __forceinline__ bool wk_unset(double v) { return __double2hiint(v) == -1; }
__device__ __forceinline__ double wk_sentinel() { return __longlong_as_double(-1LL); }
constexpr long long WK_SPIN = 4000000000LL;   // ~2 s: a missing peer -> info bit 4 instead of a hang

__device__ __forceinline__ double2 wk_ldv2(const double* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// fragments of one chunk of four pieces (8 K steps) of the T product, issue half: B = W_j rows
// of the own columns and A = had from the pieces (may still be sentinels: wk_verify_chunk).
// K step h of piece p contracts the terms 8 p + 2 t + h (t = lane % 4): a lane's two steps of
// a piece are adjacent words -> one 16-byte load each for A and B.
__device__ __forceinline__ void wk_issue_chunk(const double* pc, const double* wrow, bool wvalid, int R, int pb, int p1,
                                               double (&fa)[32], double (&fb)[8]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double* src = pc + (size_t)(pb + i) * W_PIECE + g * 8 + 2 * t;
    const bool pv = pb + i < p1;
    const int k = 8 * (pb + i) + 2 * t;
    if (pv && wvalid && k + 1 < R && !(R & 1)) {
      const double2 b = __ldg(reinterpret_cast<const double2*>(wrow + k));
      fb[2 * i] = b.x; fb[2 * i + 1] = b.y;
    } else {
      fb[2 * i] = (pv && wvalid && k < R) ? __ldg(wrow + k) : 0.0;
      fb[2 * i + 1] = (pv && wvalid && k + 1 < R) ? __ldg(wrow + k + 1) : 0.0;
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const double2 v = pv ? wk_ldv2(src + mt * 64) : make_double2(0.0, 0.0);
      fa[(2 * i) * 4 + mt] = v.x;
      fa[(2 * i + 1) * 4 + mt] = v.y;
    }
  }
}

// verify half: reload the A fragments until no word of the chunk is a sentinel
__device__ __forceinline__ void wk_verify_chunk(const double* pc, int pb, int p1, volatile int* dead, double (&fa)[32]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const long long t0 = clock64();
  for (;;) {
    bool bad = false;
#pragma unroll
    for (int q = 0; q < 32; ++q) bad |= wk_unset(fa[q]);
    if (!__any_sync(0xffffffffu, bad) || *dead) break;
    if (clock64() - t0 > WK_SPIN) { *dead = 1; break; }
    __nanosleep(64);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double* src = pc + (size_t)(pb + i) * W_PIECE + g * 8 + 2 * t;
      const bool pv = pb + i < p1;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const double2 v = pv ? wk_ldv2(src + mt * 64) : make_double2(0.0, 0.0);
        fa[(2 * i) * 4 + mt] = v.x;
        fa[(2 * i + 1) * 4 + mt] = v.y;
      }
    }
  }
}

// light wait for a warp's K range: one word of every piece [p0, p1) (lane-strided), with back-off
__device__ __forceinline__ void wk_wait_pieces(const double* pc, int p0, int p1, volatile int* dead) {
  const int lane = threadIdx.x & 31;
  const long long t0 = clock64();
  for (int p = p0 + lane; p < p1; p += 32) {
    const double* w = pc + (size_t)p * W_PIECE + W_HAD - 1;
    while (wk_unset(wk_ldv(w)) && !*dead) {
      if (clock64() - t0 > WK_SPIN) { *dead = 1; break; }
      __nanosleep(32);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void wk_mma_chunk(const double (&fa)[32], const double (&fb)[8], double (&acc)[4][2]) {
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) dmma_8x8x4(acc[mt][0], acc[mt][1], fa[ks * 4 + mt], fb[ks]);
}

// N words src[q * stride], q < n (n <= N), spun on until all are written
template <int N>
__device__ __forceinline__ void wk_ldn(const double* src, size_t stride, int n, volatile int* dead, double (&v)[N]) {
  const long long t0 = clock64();
  for (;;) {
    bool bad = false;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      v[q] = q < n ? wk_ldv(src + (size_t)q * stride) : 0.0;
      bad |= wk_unset(v[q]);
    }
    if (!bad || *dead) break;
    if (clock64() - t0 > WK_SPIN) { *dead = 1; break; }
  }
}

// one 8 x 8 tile of a (32 x 32) x (32 x 8) product, K = 32 as two interleaved chains of four steps:
// A rows at a32 (+32 bytes per step), B rows at b32 (+256 bytes per step)
__device__ __forceinline__ double2 wk_tile_k32(uint32_t a32, uint32_t b32) {
  double p0 = 0.0, p1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ks += 2) {
    dmma_8x8x4(p0, p1, lds64(a32 + 32u * (uint32_t)ks), lds64(b32 + 256u * (uint32_t)ks));
    dmma_8x8x4(q0, q1, lds64(a32 + 32u * (uint32_t)(ks + 1)), lds64(b32 + 256u * (uint32_t)(ks + 1)));
  }
  return make_double2(p0 + q0, p1 + q1);
}

#define WK_PROFT(i, T)                                                                    \
  do {                                                                                    \
    if (PROF && a.prof && (int)blockIdx.x == a.prof_cta && threadIdx.x == (T)) {          \
      const long long t_ = clock64();                                                     \
      prof_acc[i] += t_ - prof_t;                                                         \
      prof_t = t_;                                                                        \
      if (uround == 61 || uround == 62) a.prof[16 + 16 * (uround - 61) + (i)] = t_;       \
    }                                                                                     \
  } while (0)

// e-th entry (e = 32 i + c) of prod_{k != skip} G_k for the 8 entries e0 + 128 q of a thread
__device__ __forceinline__ void wk_gprod8(const WSmem& sm, int d, int skip, int e0, double (&v)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = 1.0;
  for (int k = 0; k < d; ++k) {
    if (k == skip) continue;
    const double* G = sm.Gs + (size_t)k * WK_MAT;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + 128 * q;
      v[q] *= G[(e >> 5) * WK_RH + (e & 31)];
    }
  }
}

// PROF: clock64 phase probes compiled in (debug hook; the probe code alone shifts the kernel's timing by
// several per cent through its size, so the product instantiation carries none)
// RESID: residual rounds (trace / stopping rules) compiled in.
// DC: compile-time mode count (0: a.d) -- the per-mode product loops unroll.
template <bool PROF, bool RESID, int DC>
__global__ void __launch_bounds__(WK_NT, 1) als_w(const __grid_constant__ WArgs a) {
  const bool need_resid = RESID;   // (== a.need_resid: the host picks the instantiation)
  extern __shared__ __align__(16) double smem[];
  const int d = DC ? DC : a.d, R = a.R, r = a.r, P = a.P;
  const WSmem sm = wk_carve(smem, d);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  // pair mode: the two CTAs of a cluster share a column slab and split the K range of its T product
  const int pr = a.pair, cid = blockIdx.x, NC = gridDim.x;
  const int c = cid >> pr, h = cid & pr, col0 = W_SLAB * c;
  const int wv = min(W_SLAB, R - col0);
  volatile int* dead = sm.flag + 1;
  long long prof_t = clock64(), prof_acc[16] = {};
  constexpr int PT = 128;   // profiling thread (first thread of the A group)
  constexpr size_t MSZ = (size_t)W_RM * W_RM;

  // ---- setup: zero, initial crosses / Grams of the guess, had_0, first piece
  for (size_t e = tid; e < wk_smem_doubles(d); e += WK_NT) smem[e] = 0.0;
  __syncthreads();
  // initial crosses C_k[:, own] = U_k^T V_k[:, own]: the rows of the mode split over the 8 warps
  for (int k = 0; k < d; ++k) {
    const int qk = a.q[k], r0 = (qk * warp) / 8, r1 = (qk * (warp + 1)) / 8;
    const double* Uk = a.U + a.offU[k];
    const double* Vk = a.V + a.offV[k] + col0;
    double acc[4][2] = {};
#pragma unroll 8
    for (int row = r0; row < r1; row += 4) {
      const int rr = row + t;
      const bool rv = rr < r1;
      const double fb = (rv && g < wv) ? __ldg(Vk + (size_t)rr * R + g) : 0.0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int m = 8 * mt + g;
        const double fa = (rv && m < r) ? __ldcg(Uk + (size_t)rr * r + m) : 0.0;
        dmma_8x8x4(acc[mt][0], acc[mt][1], fa, fb);
      }
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
      *reinterpret_cast<double2*>(sm.Yp + warp * W_HAD + (8 * mt + g) * 8 + 2 * t) = make_double2(acc[mt][0], acc[mt][1]);
    __syncthreads();
    {
      double v = 0.0;
      for (int w = 0; w < 8; ++w) v += sm.Yp[w * W_HAD + tid];
      sm.Cs[k * W_HAD + tid] = v;
    }
    __syncthreads();
  }
  // initial Grams G_k = U_k^T U_k: the 16 d tiles dealt to the CTAs, gathered through the armed buffer
  for (int it = cid; it < 16 * d; it += NC) {
    const int k = it >> 4, mt = (it >> 2) & 3, nt = it & 3;
    const int qk = a.q[k], r0 = (qk * warp) / 8, r1 = (qk * (warp + 1)) / 8;
    const double* Uk = a.U + a.offU[k];
    double g0 = 0.0, g1 = 0.0;
#pragma unroll 8
    for (int row = r0; row < r1; row += 4) {
      const int rr = row + t;
      const bool rv = rr < r1;
      const int m = 8 * mt + g, n = 8 * nt + g;
      const double fa = (rv && m < r) ? __ldcg(Uk + (size_t)rr * r + m) : 0.0;
      const double fb = (rv && n < r) ? __ldcg(Uk + (size_t)rr * r + n) : 0.0;
      dmma_8x8x4(g0, g1, fa, fb);
    }
    *reinterpret_cast<double2*>(sm.Yp + warp * 64 + g * 8 + 2 * t) = make_double2(g0, g1);
    __syncthreads();
    if (tid < 64) {
      double v = 0.0;
      for (int w = 0; w < 8; ++w) v += sm.Yp[w * 64 + tid];
      a.g0buf[(size_t)k * MSZ + (8 * mt + (tid >> 3)) * W_RM + 8 * nt + (tid & 7)] = v;
    }
    __syncthreads();
  }
  for (int e = tid; e < d * (int)MSZ; e += 8 * WK_NT) {
    double v[8];
    const int n = min(8, (d * (int)MSZ - e + WK_NT - 1) / WK_NT);
    wk_ldn<8>(a.g0buf + e, WK_NT, n, dead, v);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int ee = e + q * WK_NT;
      if (q < n) sm.Gs[(size_t)(ee >> 10) * WK_MAT + ((ee >> 5) & 31) * WK_RH + (ee & 31)] = v[q];
    }
  }
  __syncthreads();
  {
    double v = 1.0;
    for (int k = 1; k < d; ++k) v *= sm.Cs[k * W_HAD + tid];
    sm.hads[tid] = v;
    if (h == 0) a.pieces[((size_t)0 * P + c) * W_PIECE + tid] = v;
  }
  if (pr) {
    if (tid == 0) {
      mbar_init(sm.bar, 1);
      mbar_init(sm.bar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    wk_cluster_barrier();   // the peer is running and its barriers exist before any remote store
  }
  __syncthreads();

  int uround = 0;
  WK_PROFT(12, 0);   // setup (crosses / Grams of the guess, first piece)
  const double norm_sq = need_resid ? fmax(*a.norm_sq, 0.0) : 0.0;
  const double t_norm = sqrt(norm_sq);
  double prev = INFINITY;
  int done = 0, abort_ = 0, hb = 0, xpend = -1;   // hb: which hads buffer holds had_j of the current round
  // K range of the GEMM warps (pieces) and this CTA's share of the M entries
  const int kb0 = pr ? h * ((P + 1) / 2) : 0, kb1 = pr ? min(P, kb0 + (P + 1) / 2) : P;   // this CTA's pieces
  const int npw = (kb1 - kb0 + 3) / 4;
  const int e0 = (int)((MSZ * cid) / NC), ne = (int)((MSZ * (cid + 1)) / NC) - e0;
  int nev = 1;
  while (nev < ne) nev <<= 1;
  const int ngr = 128 / nev;                 // producer groups of the Gram reduction (A group, 128 threads)
  const int ppg = (P + ngr - 1) / ngr;       // producers per group

  for (int sweep = 0;; ++sweep) {
    bool stop = false;
    for (int j = 0; j < d; ++j) {
      const bool first = sweep == 0 && j == 0;
      const int slot = (sweep & 1) * d + j;
      const double* pc = a.pieces + (size_t)slot * P * W_PIECE;
      const int jp = (j + d - 1) % d;
      const bool last_half = sweep == a.sweeps;   // only the residual of the last sweep is still due
      const bool resid_round = need_resid && j == 0 && sweep > 0;
      // the previous round's Newton-Schulz update X_xp = X0 Tn_prev is still pending: the reducers
      // apply it as two vector products, warps 0-3 form the matrix while they wait at the join
      const int xp = xpend;
      double* Tcur = sm.Tn + (size_t)(uround & 1) * WK_MAT;
      const double* Tprev = sm.Tn + (size_t)((uround & 1) ^ 1) * WK_MAT;
      if (last_half && !need_resid) { stop = true; break; }
      WK_PROFT(0, PT);
      // ---- A group, part 1: reduce the partial Grams of update jp, G_jp = sym(sum)
      if (warp >= 4 && !first) {
        const int t2 = tid - 128;
        double* ms = a.msum + (size_t)slot * MSZ;
        {
          // this CTA's entries [e0, e0 + ne) of the summed partial Grams: group grp sums its
          // producers in order, then the groups in order
          const int ei = t2 & (nev - 1), grp = t2 / nev;
          double s = 0.0;
          if (ei < ne) {
            const int pa = grp * ppg, pb = min(P, pa + ppg);
            for (int p = pa; p < pb; p += 8) {
              double v[8];
              wk_ldn<8>(pc + (size_t)p * W_PIECE + W_HAD + e0 + ei, W_PIECE, pb - p, dead, v);
#pragma unroll
              for (int q = 0; q < 8; ++q) s += v[q];
            }
          }
          sm.red[t2] = s;
          wk_bar(1, 128);
          if (t2 < ne) {
            double tot = 0.0;
            for (int gi = 0; gi < ngr; ++gi) tot += sm.red[gi * nev + t2];
            ms[e0 + t2] = tot;
            a.msum[(size_t)(slot < d ? slot + d : slot - d) * MSZ + e0 + t2] = wk_sentinel();   // re-arm the other parity
          }
        }
        WK_PROFT(1, PT);
        {
          double v[8];
          wk_ldn<8>(ms + t2, 128, 8, dead, v);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int e = t2 + 128 * q;
            sm.Ms[(e >> 5) * WK_RH + (e & 31)] = v[q];
          }
        }
        wk_bar(1, 128);
        WK_PROFT(2, PT);
        double* Gj = sm.Gs + (size_t)jp * WK_MAT;   // G_jp = sym(M X_jp)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = t2 + 128 * q, i = e >> 5, cc = e & 31;
          Gj[i * WK_RH + cc] = 0.5 * (sm.Ms[i * WK_RH + cc] + sm.Ms[cc * WK_RH + i]);
        }
        wk_bar(1, 128);
        WK_PROFT(3, PT);
      }
      // ---- residual of the finished sweep (Gram identity, cp.py:321-326) and stopping rules
      if (resid_round) {
        __syncthreads();
        double ov = 0.0;
        for (int p = 0; p < P; p += 8) {
          double v[8];
          wk_ldn<8>(pc + (size_t)p * W_PIECE + W_HAD + MSZ, W_PIECE, P - p, dead, v);
#pragma unroll
          for (int q = 0; q < 8; ++q) ov += v[q];
        }
        double sv = 0.0;
        for (int e = tid; e < W_RM * W_RM; e += WK_NT) {
          const int i = e >> 5, cc = e & 31;
          double v = 1.0;
          for (int k = 0; k < d; ++k) v *= sm.Gs[(size_t)k * WK_MAT + i * WK_RH + cc];
          if (i < r && cc < r) sv += v;
        }
        const double self = wk_block_sum(sv, sm.red);
        const double resid = sqrt(fmax(norm_sq - 2.0 * ov + self, 0.0));
        if (cid == 0 && tid == 0 && a.trace) a.trace[sweep - 1] = resid;
        if (resid <= a.tol * t_norm) stop = true;
        if (prev - resid < a.stall * fmax(t_norm, 1.0)) stop = true;
        prev = resid;
      }
      if (last_half) stop = true;
      if (stop) break;
      if (warp >= 4) {
        // ---- A group, part 2: A_j = prod_{k != j} G_k + lambda I (cp.py:171-173, 312-315) and the
        // Newton-Schulz residual of the previous sweep's X_j: Tn = 2I - A_j X_j, |I - A_j X_j|
        const int t2 = tid - 128;
        double lam = a.reg;
        if (a.reg_mode) {
          double tr = 0.0;
          for (int i = 0; i < r; ++i) {
            double v = 1.0;
            for (int k = 0; k < d; ++k)
              if (k != j) v *= sm.Gs[(size_t)k * WK_MAT + i * WK_RH + i];
            tr += v;
          }
          lam = a.reg * fmax(tr, 0.0) / (double)r;
        }
        {
          double v[8];
          wk_gprod8(sm, d, j, t2, v);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int e = t2 + 128 * q, i = e >> 5, cc = e & 31;
            sm.Am[i * WK_RH + cc] = (i < r && cc < r) ? v[q] + (i == cc ? lam : 0.0) : 0.0;
          }
        }
        wk_bar(1, 128);
        int ok = 0;
        if (sweep > 0) {
          double em = wk_gemm32(sm.Am, sm.Xs + (size_t)j * WK_MAT, Tcur, r, 0, 4);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
          if (lane == 0) sm.part[warp - 4] = em;
          wk_bar(1, 128);
          em = fmax(fmax(sm.part[0], sm.part[1]), fmax(sm.part[2], sm.part[3]));
          ok = em <= 1e-8;   // (NaN fails); one step squares the error: |I - A X1| <= (r 1e-8)^2
        }
        // no warm start / rejected: the exact inverse on these four warps, still beside the T product
        // (flag 1: Newton-Schulz accepted, 2: exact X_j in place, 3: ill-conditioned -> fallback)
        if (!ok) {
          double ratio;
          wk_inverse(sm, r, sm.Xs + (size_t)j * WK_MAT, &ratio);
          ok = (ratio <= a.cond_max) ? 2 : 3;
        }
        if (tid == 128) sm.flag[0] = ok;
        WK_PROFT(4, PT);
      } else {
        // ---- GEMM group: T_j[:, own] = had_j W_j[:, own], K split over the four warps
        const int p0 = kb0 + warp * npw, p1 = min(kb1, p0 + npw);
        const int nch = (max(p1 - p0, 0) + 3) / 4;
        const bool wvalid = g < wv;
        const double* wrow = a.W + (size_t)j * R * R + (size_t)(col0 + (wvalid ? g : 0)) * R;
        double acc[4][2] = {};
        double fa0[32], fb0[8], fa1[32], fb1[8];
        wk_wait_pieces(pc, p0, p1, dead);
        if (nch > 0) wk_issue_chunk(pc, wrow, wvalid, R, p0, p1, fa0, fb0);
        for (int ch = 0; ch < nch; ch += 2) {
          if (ch + 1 < nch) wk_issue_chunk(pc, wrow, wvalid, R, p0 + 4 * (ch + 1), p1, fa1, fb1);
          wk_verify_chunk(pc, p0 + 4 * ch, p1, dead, fa0);
          wk_mma_chunk(fa0, fb0, acc);
          if (ch + 2 < nch) wk_issue_chunk(pc, wrow, wvalid, R, p0 + 4 * (ch + 2), p1, fa0, fb0);
          if (ch + 1 < nch) {
            wk_verify_chunk(pc, p0 + 4 * (ch + 1), p1, dead, fa1);
            wk_mma_chunk(fa1, fb1, acc);
          }
        }
        WK_PROFT(8, 0);
        double* tp = sm.Tp + warp * W_HAD;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
          *reinterpret_cast<double2*>(tp + (8 * mt + g) * 8 + 2 * t) = make_double2(acc[mt][0], acc[mt][1]);
        wk_bar(2, 128);
        double* tsum = pr ? sm.Tl : sm.Ts;
        for (int e = tid; e < W_HAD; e += 128)
          tsum[e] = (sm.Tp[e] + sm.Tp[W_HAD + e]) + (sm.Tp[2 * W_HAD + e] + sm.Tp[3 * W_HAD + e]);
        if (pr) {
          // the other half of the K range comes from the peer: each CTA pushes its partial into the
          // peer's buffer (st.async onto the peer's mbarrier) and adds in rank order
          const int par = uround & 1;
          wk_bar(2, 128);
          if (tid == 0) mbar_arrive_expect_tx(sm.bar + par, (uint32_t)(W_HAD * sizeof(double)));
          const uint32_t dst = mapa_u32(smem_u32(sm.Tx + par * W_HAD), (uint32_t)(h ^ 1));
          const uint32_t rbar = mapa_u32(smem_u32(sm.bar + par), (uint32_t)(h ^ 1));
          wk_st_async_v2(dst + 16u * (uint32_t)tid, sm.Tl[2 * tid], sm.Tl[2 * tid + 1], rbar);
          mbar_wait(sm.bar + par, (uint32_t)((uround >> 1) & 1));
          const double* tx = sm.Tx + par * W_HAD;
          for (int e = tid; e < W_HAD; e += 128) sm.Ts[e] = h == 0 ? sm.Tl[e] + tx[e] : tx[e] + sm.Tl[e];
        }
        if (xp >= 0) wk_gemm32(sm.Xs + (size_t)xp * WK_MAT, Tprev, sm.X1, r, 1, 0);   // X1 = X0 (2I - A X0)
      }
      WK_PROFT(9, 0);
      __syncthreads();
      WK_PROFT(10, 0);
      WK_PROFT(5, PT);
      double* Xj = sm.Xs + (size_t)j * WK_MAT;
      if (sm.flag[0] == 3) { abort_ = 1; stop = true; break; }
      const int ok = sm.flag[0] == 1;
      WK_PROFT(6, PT);
      // ---- C_j[:, own] = X_j T_j (cp.py:316-320 in Gram space).  Warm: X_j = X0 Tn is applied
      // as X0 (Tn T_j) on warps 0-3 while warps 4-7 form the matrix X0 Tn for the next sweep
      if (warp < 4) {
        const int mt = warp;
        const uint32_t tb = smem_u32(ok ? sm.Yp : sm.Ts) + 8u * (uint32_t)(t * 8 + g);
        if (ok) {
          const uint32_t na = smem_u32(Tcur) + 8u * (uint32_t)((8 * mt + g) * WK_RH + t);
          const uint32_t sb = smem_u32(sm.Ts) + 8u * (uint32_t)(t * 8 + g);
          *reinterpret_cast<double2*>(sm.Yp + (8 * mt + g) * 8 + 2 * t) = wk_tile_k32(na, sb);
          wk_bar(2, 128);
        }
        const uint32_t xa = smem_u32(Xj) + 8u * (uint32_t)((8 * mt + g) * WK_RH + t);
        *reinterpret_cast<double2*>(sm.Cs + j * W_HAD + (8 * mt + g) * 8 + 2 * t) = wk_tile_k32(xa, tb);
      } else {
        // warps 4-7: Y = X_j had_j[:, own] (the partial Gram of this CTA is C_j[:, own] Y^T: the
        // producers publish partials of G_j = C_j had_j^T X_j itself, no product after the reduction)
        const int mt = warp - 4;
        const double* hj = sm.hads + hb * W_HAD;
        const uint32_t hb32 = smem_u32(ok ? sm.Yp + W_HAD : hj) + 8u * (uint32_t)(t * 8 + g);
        if (ok) {
          const uint32_t na = smem_u32(Tcur) + 8u * (uint32_t)((8 * mt + g) * WK_RH + t);
          const uint32_t sb = smem_u32(hj) + 8u * (uint32_t)(t * 8 + g);
          *reinterpret_cast<double2*>(sm.Yp + W_HAD + (8 * mt + g) * 8 + 2 * t) = wk_tile_k32(na, sb);
          wk_bar(1, 128);
        }
        const uint32_t xa = smem_u32(Xj) + 8u * (uint32_t)((8 * mt + g) * WK_RH + t);
        *reinterpret_cast<double2*>(sm.Yp + 2 * W_HAD + (8 * mt + g) * 8 + 2 * t) = wk_tile_k32(xa, hb32);
        if (xp >= 0) {
          double* Xp = sm.Xs + (size_t)xp * WK_MAT;
          for (int e = tid - 128; e < WK_MAT; e += 128) Xp[e] = sm.X1[e];
        }
      }
      __syncthreads();
      xpend = ok ? j : -1;   // the matrix X_j = X0 Tn is formed during the next round
      // ---- this CTA's piece of the next round: partial Gram C_j[:, own] Y^T, own columns of had_{j+1}
      const int jn = (j + 1) % d;
      const int nsweep = sweep + (jn == 0 ? 1 : 0);
      const bool publish = need_resid || nsweep < a.sweeps;
      if (publish) {
        double* pn = a.pieces + ((size_t)((nsweep & 1) * d + jn) * P + c) * W_PIECE;
        const double* yj = sm.Yp + 2 * W_HAD;
        {
          double v = 1.0;
          for (int k = 0; k < d; ++k)
            if (k != jn) v *= sm.Cs[k * W_HAD + tid];
          sm.hads[(hb ^ 1) * W_HAD + tid] = v;
          if (h == 0) pn[tid] = v;
        }
        for (int tile = warp; tile < 16; tile += 8) {
          const int mt = tile >> 2, nt = tile & 3;
          double m0 = 0.0, m1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            dmma_8x8x4(m0, m1, sm.Cs[j * W_HAD + (8 * mt + g) * 8 + 4 * ks + t], yj[(8 * nt + g) * 8 + 4 * ks + t]);
          if (h == 0) *reinterpret_cast<double2*>(pn + W_HAD + (8 * mt + g) * W_RM + 8 * nt + 2 * t) = make_double2(m0, m1);
        }
        if (need_resid && j == d - 1) {
          double v = 1.0;
          for (int k = 0; k < d; ++k) v *= sm.Cs[k * W_HAD + tid];
          const double ov = wk_block_sum(v, sm.red);
          if (tid == 0 && h == 0) pn[W_HAD + MSZ] = ov;
        }
        // re-arm this CTA's piece of mode j, previous sweep (every reader finished it a sweep ago;
        // its next use is the sweep after this one)
        if (sweep >= 1 && h == 0) {
          double* po = a.pieces + ((size_t)(((sweep - 1) & 1) * d + j) * P + c) * W_PIECE;
          for (int e = tid; e < W_PIECE; e += WK_NT) po[e] = wk_sentinel();
        }
        hb ^= 1;
        // (every shared buffer written before the next join is disjoint from what slower warps
        // still read here, except the block-sum scratch of the residual rounds)
        if (need_resid) __syncthreads();
      }
      WK_PROFT(7, PT);
      WK_PROFT(11, 0);
      ++uround;
    }
    if (stop) { done = sweep; break; }
  }

  WK_PROFT(13, 0);   // (tail of the last round)
  // ---- after the last sweep: U_j = V_j had_j^T X_j (had_j of the last update of mode j)
  if (!abort_ && done > 0) {
    __syncthreads();
    if (xpend >= 0) {   // the last Newton-Schulz matrix update
      double* Xp = sm.Xs + (size_t)xpend * WK_MAT;
      if (warp < 4) wk_gemm32(Xp, sm.Tn + (size_t)((uround & 1) ^ 1) * WK_MAT, sm.X1, r, 1, 0);
      __syncthreads();
      for (int e = tid; e < WK_MAT; e += WK_NT) Xp[e] = sm.X1[e];
      __syncthreads();
    }
    const int ls = done - 1;
    int nf = 0;
    for (int it = cid; it < a.tile0[d]; it += NC) {
      int j = 0;
      while (it >= a.tile0[j + 1]) ++j;
      const int row0 = 8 * (it - a.tile0[j]), qj = a.q[j];
      const double* pc = a.pieces + (size_t)((ls & 1) * d + j) * P * W_PIECE;
      const double* vrow = a.V + a.offV[j] + (size_t)min(row0 + g, qj - 1) * R;
      const bool rv = row0 + g < qj;
      double acc[4][2] = {};
      const int pp0 = (P * warp) / 8, pp1 = (P * (warp + 1)) / 8;
#pragma unroll 2
      for (int p = pp0; p < pp1; ++p) {
        const double* src = pc + (size_t)p * W_PIECE + g * 8 + t;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = 8 * p + 4 * h + t;
          const double fa = (rv && k < R) ? __ldg(vrow + k) : 0.0;
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[nt][0], acc[nt][1], fa, __ldcg(src + nt * 64 + 4 * h));
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        *reinterpret_cast<double2*>(sm.Yp + warp * W_HAD + g * W_RM + 8 * nt + 2 * t) = make_double2(acc[nt][0], acc[nt][1]);
      __syncthreads();
      {
        double v = 0.0;
        for (int w = 0; w < 8; ++w) v += sm.Yp[w * W_HAD + tid];
        sm.Ys[(tid >> 5) * WK_RH + (tid & 31)] = v;
      }
      __syncthreads();
      if (warp < 4) {
        const int nt = warp;
        double u0 = 0.0, u1 = 0.0;
        const double* Xj = sm.Xs + (size_t)j * WK_MAT;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          dmma_8x8x4(u0, u1, sm.Ys[g * WK_RH + 4 * ks + t], Xj[(4 * ks + t) * WK_RH + 8 * nt + g]);
        const int row = row0 + g, i0 = 8 * nt + 2 * t;
        if (row < qj) {
          double* dst = a.U + a.offU[j] + (size_t)row * r;
          if (i0 < r) { dst[i0] = u0; if (!isfinite(u0)) nf = 1; }
          if (i0 + 1 < r) { dst[i0 + 1] = u1; if (!isfinite(u1)) nf = 1; }
        }
      }
      __syncthreads();
    }
    if (nf) atomicOr(a.info, 2);
  }
  WK_PROFT(14, 0);   // final phase
  if (tid == 0) {
    if (*dead) atomicOr(a.info, 4);
    if (cid == 0) {
      if (abort_) *a.redo = 1;
      else a.info[1] = done;
    }
  }
  if (PROF && a.prof && (int)blockIdx.x == a.prof_cta && (tid == PT || tid == 0))
    for (int q = (tid == 0 ? 8 : 0); q < (tid == 0 ? 16 : 8); ++q) a.prof[q] += prof_acc[q];
  if (pr) {
    __syncthreads();
    wk_cluster_barrier();   // no CTA exits while its peer may still store into its shared memory
  }
}

// product instantiations: the usual mode counts compiled in (config 1: 827 -> 781 us per truncation with
// d = 6 a constant), any other through the generic one
template <bool RESID>
static const void* wk_kernel(int d) {
  switch (d) {
    case 3: return (const void*)als_w<false, RESID, 3>;
    case 4: return (const void*)als_w<false, RESID, 4>;
    case 5: return (const void*)als_w<false, RESID, 5>;
    case 6: return (const void*)als_w<false, RESID, 6>;
    default: return (const void*)als_w<false, RESID, 0>;
  }
}

static int g_w_pair = 1;          // debug hook: 0 = one CTA per column slab (no K split over a CTA pair)
static int g_w_on = 1;            // debug hook: 0 = never plan the Gram-space kernel
static double g_w_cond = 1e3;     // debug hook: pivot-ratio bound above which the direct kernel reruns

int als_w_enabled() { return g_w_on + 2 * g_w_pair; }

int als_w_plan(int d, const int* q, int R, int r, WPlan& pl) {
  if (!g_w_on || d < 2 || d > TP_MAXD || r < 1 || r > W_RM || R < 1) return TP_EUNSUPPORTED;
  const int P = (R + W_SLAB - 1) / W_SLAB;
  int dev = 0, nsm = 148, smem_optin = 227 * 1024;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  } else {
    cudaGetLastError();
  }
  if (P < 32 || P > nsm) return TP_EUNSUPPORTED;   // (the reducer shares need <= 32 entries per CTA)
  int qmin = q[0], qmax = q[0];
  for (int k = 0; k < d; ++k) { qmin = q[k] < qmin ? q[k] : qmin; qmax = q[k] > qmax ? q[k] : qmax; }
  if (4 * qmin < R) return TP_EUNSUPPORTED;        // R^2 work per update instead of Q R: only for R <~ Q
  WArgs& a = pl.a;
  memset(&a, 0, sizeof(a));
  a.d = d; a.R = R; a.r = r; a.P = P;
  a.pair = (g_w_pair && 2 * P <= nsm) ? 1 : 0;
  long long ov = 0, ou = 0;
  int tiles = 0;
  for (int k = 0; k < d; ++k) {
    a.q[k] = q[k]; a.offV[k] = ov; a.offU[k] = ou; a.tile0[k] = tiles;
    ov += (long long)q[k] * R; ou += (long long)q[k] * r; tiles += (q[k] + 7) / 8;
  }
  a.tile0[d] = tiles;
  pl.uniform_q = qmin == qmax;
  pl.smem = wk_smem_doubles(d) * sizeof(double);
  if (pl.smem > (size_t)smem_optin) return TP_EUNSUPPORTED;
  if (a.pair) {   // P co-resident 2-CTA clusters?
    cudaFuncSetAttribute(als_w<false, false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    cudaGetLastError();
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * P); cfg.blockDim = dim3(WK_NT); cfg.dynamicSmemBytes = pl.smem;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nclu = 0;
    if (cudaOccupancyMaxActiveClusters(&nclu, (const void*)als_w<false, false, 0>, &cfg) != cudaSuccess) { cudaGetLastError(); nclu = 0; }
    if (nclu < P) a.pair = 0;
  }
  pl.ws_inner = align_up(sizeof(double) * (size_t)inner_tiles(R, R, 1));
  pl.ws = align_up(sizeof(double) * (size_t)d * R * R) + align_up(sizeof(double) * 2 * (size_t)d * P * W_PIECE) +
          align_up(sizeof(double) * 3 * (size_t)d * W_RM * W_RM) + 512 + align_up(sizeof(int)) + align_up(sizeof(double)) +
          pl.ws_inner + 256;
  return TP_OK;
}

int als_w_run(const WPlan& plan, const double* V, double* U, int sweeps, double reg, int reg_mode, double tol,
              double stall, double* trace, int* info, void* ws, size_t ws_bytes, cudaStream_t st, long long* prof,
              int prof_cta, const int** redo_out) {
  if (!ws || ws_bytes < plan.ws) return TP_EWORKSPACE;
  WArgs a = plan.a;
  const int d = a.d, R = a.R, P = a.P;
  Carver cv(ws, ws_bytes);
  double* W = cv.take<double>((size_t)d * R * R);
  a.pieces = cv.take<double>(2 * (size_t)d * P * W_PIECE);   // pieces, msum: one memset to the sentinel
  a.msum = cv.take<double>(2 * (size_t)d * W_RM * W_RM);
  a.g0buf = cv.take<double>((size_t)d * W_RM * W_RM);
  a.redo = cv.take<int>(1);
  double* nsq = cv.take<double>(1);
  double* part = cv.take<double>(plan.ws_inner / sizeof(double));
  a.W = W;
  a.V = V; a.U = U; a.trace = trace; a.info = info; a.norm_sq = nsq;
  a.sweeps = sweeps; a.reg = reg; a.reg_mode = reg_mode; a.tol = tol; a.stall = stall;
  a.need_resid = (trace != nullptr) || (tol > 0.0) || (stall > -INFINITY);
  a.cond_max = g_w_cond;
  a.prof = prof; a.prof_cta = prof_cta;
  *redo_out = a.redo;
  cudaError_t e = cudaMemsetAsync(info, 0, 2 * sizeof(int), st);
  if (e != cudaSuccess) return cuda_status(e);
  e = cudaMemsetAsync(a.redo, 0, sizeof(int), st);
  if (e != cudaSuccess) return cuda_status(e);
  if (sweeps == 0) return TP_OK;
  // exchange buffers armed: all-ones words = "not written yet"
  e = cudaMemsetAsync(a.pieces, 0xFF, (size_t)(reinterpret_cast<char*>(a.redo) - reinterpret_cast<char*>(a.pieces)), st);
  if (e != cudaSuccess) return cuda_status(e);
  if (sweeps == 0) return TP_OK;
  if (a.need_resid) {
    const int s = launch_inner(d, a.q, R, V, R, V, 1, nsq, part, st);   // ||V||^2 (cp.py:186-188)
    if (s != TP_OK) return s;
  }
  // W_k = V_k^T V_k (batched over the modes when the grids agree)
  const int nbat = plan.uniform_q ? 1 : d;
  for (int b = 0; b < nbat; ++b) {
    const int qk = a.q[b];
    const double* Vk = V + a.offV[b];
    BGemm gw = bgemm_desc(R, R, qk, Vk, 1, R, Vk, R, 1, W + (size_t)b * R * R, R, 1);
    if (plan.uniform_q) {
      gw.nb1 = d;
      gw.sA1 = gw.sB1 = (long long)qk * R; gw.sC1 = (long long)R * R;
    }
    e = bgemm_launch(gw, st);
    if (e != cudaSuccess) return cuda_status(e);
  }
  const void* fn = prof ? (a.need_resid ? (const void*)als_w<true, true, 0> : (const void*)als_w<true, false, 0>)
                        : (a.need_resid ? wk_kernel<true>(d) : wk_kernel<false>(d));
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
  if (e != cudaSuccess) return cuda_status(e);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.pair ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.gridDim = dim3(P << a.pair); cfg.blockDim = dim3(WK_NT); cfg.dynamicSmemBytes = plan.smem; cfg.stream = st;
  cfg.attrs = at; cfg.numAttrs = 2;
  static const bool noncoop = getenv("TP_ALS_NONCOOP") && getenv("TP_ALS_NONCOOP")[0] == '1';
  if (noncoop) cfg.numAttrs = 1;
  void* args[] = {&a};
  return cuda_status(cudaLaunchKernelExC(&cfg, fn, args));
}

}  // namespace tp

extern "C" void tp_debug_set_als_w_pair(int on) { tp::g_w_pair = on; }
extern "C" void tp_debug_set_als_w(int on, double cond_max) {
  tp::g_w_on = on;
  if (cond_max > 0.0) tp::g_w_cond = cond_max;
}
