// Cluster-row CP-ALS (cp.cp_approx_als, cp.py:266-334) for large truncations
// (BASELINE config 1: d=6, Q=256, R=512, r=32): one launch runs every sweep.
//
// Grid = P clusters x S CTAs (S = 16, non-portable cluster size).  Cluster c owns
// the R-slab [c0, c1) of the target terms; CTA b of a cluster owns row block b of
// every mode (rows [Q_k b / S, Q_k (b+1) / S)) and keeps V_k[block, slab] for
// all k in shared memory.  Every cluster solves ALL rows of the iterate
// redundantly: CTA b of cluster c computes U_j[block b] itself, so the only
// cross-cluster exchange of a mode update is the right-hand-side reduction
// among the P CTAs that own the same row block -- flag-synchronised through L2,
// no grid barrier.  A mode update j (cp.py:311-320):
//
//  1. Y_cb = V_j[block b, slab c] had_j^T   (partial rhs, DMMA, K = slab columns)
//     -> global slot (c, b); release flag.  While the peers' slots land:
//     A_j = prod_{k!=j} G_k + lambda I (cp.py:171-173) and A_j^-1 by the
//     symmetric sweep operator (every CTA, identical).
//  2. acquire the P flags of row block b; rhs = sum_c Y_cb (fixed order c = 0..P-1,
//     bitwise identical in every cluster); U_j[block b] = rhs A_j^-1 (DMMA).
//  3. cluster exchange for mode j: CTA b forms the partial cross U_j[blk]^T V_j[blk,
//     slab] and partial Gram U_j[blk]^T U_j[blk] (DMMA) and stores each element
//     straight into its owner's inbox (st.shared::cluster; CTA o owns slab columns
//     [w o / S, w (o+1) / S) and Gram entries [r^2 o / S, r^2 (o+1) / S));
//     cluster barrier; the owner sums the S partials in rank order, keeps its
//     columns of C_j (and of every C_k), forms its columns of
//     had_{j+1} = prod_{k!=j+1} C_k (cp.py:197-201) and stores them, with its Gram
//     entries, into every CTA's had / G arrays; cluster barrier.
//
// Per mode update: two hardware cluster barriers and one P-way flag exchange
// instead of two grid barriers.  Results are bitwise reproducible for a fixed
// (P, S) (fixed summation orders everywhere).  After a sweep (only with a trace
// or a stopping rule) the residual by the Gram identity (cp.py:321-326) uses the
// overlap sum over the owners' columns (one more flag round); the stopping
// decision is identical in every CTA.
#include "tp_common.cuh"
#include "tp_als_rows.cuh"
#include <cfloat>
#include <cmath>
#include <cstring>

namespace tp {

int launch_inner(int d, const int* q, int ra, const double* A, int rb, const double* B, int same,
                 double* out, double* partial, cudaStream_t st);
int inner_tiles(int ra, int rb, int same);

constexpr int RW_NT = 256;
constexpr int RW_NW = RW_NT / 32;
constexpr int RW_PART = 512;
constexpr int RW_PMAX = 16;   // max clusters (R-slabs)

__host__ __device__ inline int rw_pad4(int n) { return n + (((4 - n % 16) + 16) % 16); }

struct RwSmem {
  double *Vs, *hadT, *Cown, *Gown, *Apk, *inbox, *Us, *Am, *X0, *X1, *scr, *rb, *gpub, *part, *pub, *scal;
  uint64_t* bar;   // [0]: warm-start prefetch, [1]: inbox (partials), [2]: publishes
  // integer tables (no runtime divisions in the hot loops)
  int* gposT;      // [r][r]: owner-major packed position of Gram entry (i, c)
  int* divT;       // [tbl]: (e / r) | (e % r) << 16
  int* nbT;        // [d]: rows of this CTA's block of mode k
  int* qb0T;       // [d]: first row of the block
  int* ocT;        // [S + 1]: first slab column owned by rank q
  int* gdiag;      // [gstride]: 1 where this rank's packed Gram entry is diagonal
};

// region sizes rounded to even doubles: every region starts 16-byte aligned (v2 / bulk copies)
__host__ __device__ inline size_t rw_ev(size_t n) { return (n + 1) & ~(size_t)1; }
__host__ __device__ inline int rw_nbr(const RowsArgs& a) { return (a.nb4max + 7) & ~7; }   // Us / rb rows
__host__ __device__ inline int rw_tbl(const RowsArgs& a) {
  int m = a.wcol > rw_nbr(a) ? a.wcol : rw_nbr(a);
  if (m < a.r) m = a.r;
  return m * a.r;
}
__host__ __device__ inline size_t rw_int_doubles(const RowsArgs& a) {
  return rw_ev((size_t)(a.r * a.r + rw_tbl(a) + 2 * TP_MAXD + a.S + 1 + a.gstride + 1) / 2 + 1);
}


// scratch, reused by phase: exchange staging (C^T partial [0, cst_len), Gram blocks after it);
// split-K partials of the rhs product [0, ysplit); Newton-Schulz temporary [0, RM rh);
// the prefetched warm start X0 at [x0off, x0off + RM rh) (lands during the rhs product)
__host__ __device__ inline size_t rw_x0off(int RM, int r) {
  const size_t y = (size_t)RW_NW * (RM / 8) * 64, t = (size_t)RM * rw_pad4(r);
  return rw_ev(y > t ? y : t);
}
__host__ __device__ inline size_t rw_scr_doubles(const RowsArgs& a, int RM) {
  const size_t x = (size_t)a.cst_len + (size_t)a.S * a.gstride;
  const size_t z = rw_x0off(RM, a.r) + (size_t)RM * rw_pad4(a.r);
  const size_t g = (size_t)a.P * rw_ev((size_t)rw_nbr(a) * a.r);   // the P gathered rhs slots
  const size_t m = x > z ? x : z;
  return m > g ? m : g;
}

__host__ __device__ inline size_t rw_smem_doubles(const RowsArgs& a, int RM) {
  const size_t rh = rw_pad4(a.r);
  return 4 + rw_int_doubles(a) + rw_ev(a.vtot) + rw_ev((size_t)a.kpad * rh) + rw_ev((size_t)a.d * a.wcol * a.r) +
         rw_ev((size_t)a.d * a.gstride) + rw_ev((size_t)a.S * a.gstride) + rw_ev((size_t)a.S * a.piece) + rw_ev((size_t)rw_nbr(a) * rh) +
         2 * rw_ev((size_t)RM * rh) + rw_ev(rw_scr_doubles(a, RM)) + rw_ev((size_t)rw_nbr(a) * rh) +
         rw_ev(a.gstride) + RW_PART + 80 + 8;
}

__device__ inline RwSmem rw_carve(double* base, const RowsArgs& a, int RM) {
  const size_t rh = rw_pad4(a.r);
  RwSmem s;
  size_t o = 0;
  s.bar = reinterpret_cast<uint64_t*>(base); o += 4;
  {
    int* ip = reinterpret_cast<int*>(base + o);
    s.gposT = ip; ip += a.r * a.r;
    s.divT = ip; ip += rw_tbl(a);
    s.nbT = ip; ip += TP_MAXD;
    s.qb0T = ip; ip += TP_MAXD;
    s.ocT = ip; ip += a.S + 1;
    s.gdiag = ip;
    o += rw_int_doubles(a);
  }
  s.Vs = base + o; o += rw_ev(a.vtot);
  s.hadT = base + o; o += rw_ev((size_t)a.kpad * rh);
  s.Cown = base + o; o += rw_ev((size_t)a.d * a.wcol * a.r);
  s.Gown = base + o; o += rw_ev((size_t)a.d * a.gstride);
  s.Apk = base + o; o += rw_ev((size_t)a.S * a.gstride);
  s.inbox = base + o; o += rw_ev((size_t)a.S * a.piece);
  s.Us = base + o; o += rw_ev((size_t)rw_nbr(a) * rh);
  s.Am = base + o; o += rw_ev((size_t)RM * rh);
  s.X1 = base + o; o += rw_ev((size_t)RM * rh);
  s.scr = base + o; o += rw_ev(rw_scr_doubles(a, RM));
  s.X0 = s.scr + rw_x0off(RM, a.r);
  s.rb = base + o; o += rw_ev((size_t)rw_nbr(a) * rh);
  s.gpub = base + o; o += rw_ev(a.gstride);
  s.part = base + o; o += RW_PART;
  s.pub = base + o; o += 80;
  s.scal = base + o;
  return s;
}

__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_v2(uint32_t addr, double x, double y) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(x), "d"(y) : "memory");
}

__device__ __forceinline__ void sts64(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double2 lds2x64(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// remote stores that complete bytes on the receiver's mbarrier (point-to-point, no barrier)
__device__ __forceinline__ void st_async_v2(uint32_t addr, double x, double y, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
               "d"(x), "d"(y), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t addr, double x, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(addr), "d"(x),
               "r"(rbar)
               : "memory");
}

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

// named barrier over the first n threads (n a multiple of 32)
__device__ __forceinline__ void bar_named(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// deterministic block sum (all threads call; result valid in all threads)
__device__ inline double rw_block_sum(double v, double* red) {
  const int tid = threadIdx.x;
  red[tid] = v;
  __syncthreads();
  for (int w = RW_NT / 2; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

// A_j -> Am (row stride rh, zero padded) from the owners' published packed blocks
// (A_j = prod_{k != j} G_k, formed by each Gram owner, cp.py:312-315) plus lambda I
// (cp.py:171-173: fixed lambda, or reg * max(tr A, 0) / r); threads [t0, t0 + nt),
// named barrier 1
__device__ void rw_build_a_w(const RowsArgs& a, const RwSmem& sm, int nt, int t0 = 0) {
  const int r = a.r, rh = rw_pad4(r), tid = threadIdx.x - t0;
  double lam = a.reg;
  if (a.reg_mode) {
    double tr = 0.0;   // (fixed order: every thread sums the diagonal itself)
    for (int i = 0; i < r; ++i) tr += sm.Apk[sm.gposT[i * r + i]];
    lam = a.reg * fmax(tr, 0.0) / (double)r;
  }
  for (int e = tid; e < r * r; e += nt) {
    const int dv = sm.divT[e], i = dv & 0xffff, c = dv >> 16;
    sts64(smem_u32(sm.Am) + 8u * (uint32_t)(i * rh + c), lds64(smem_u32(sm.Apk) + 8u * (uint32_t)sm.gposT[e]) + (i == c ? lam : 0.0));
  }
  bar_named(1, nt);
}

// lambda of the regularised normal equations (cp.py:171-173): fixed, or reg * max(tr A, 0) / r
// with the trace summed in a fixed order by every calling thread
__device__ __forceinline__ double rw_lambda(const RowsArgs& a, const RwSmem& sm) {
  if (!a.reg_mode) return a.reg;
  double tr = 0.0;
  for (int i = 0; i < a.r; ++i) tr += sm.Apk[sm.gposT[i * a.r + i]];
  return a.reg * fmax(tr, 0.0) / (double)a.r;
}

// Newton-Schulz residual step on four warps [w0, w0 + 4) for RM = 32, reading A_j + lambda I
// straight from the owners' packed blocks (fragment (i, k) at Apk[gposT[i r + k]], zero
// outside r x r): out = 2I - (A + lambda I) X, returns this thread's max |I - (A + lambda I) X|.
// Warp w owns the 2 x 2 block of 8 x 8 tiles (2 (w / 2) + {0, 1}, 2 (w % 2) + {0, 1}).
__device__ double rw_ns_packed(const RowsArgs& a, const RwSmem& sm, double lam, const double* X, double* out, int w0) {
  constexpr int RM = 32;
  const int r = a.r, rh = rw_pad4(r);
  const int warp = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
  const uint32_t apk32 = smem_u32(sm.Apk), x32 = smem_u32(X), o32 = smem_u32(out);
  const int bm = 2 * (warp >> 1), bn = 2 * (warp & 1);
  double acc[2][2][2] = {};
  const uint32_t bc = x32 + 8u * (uint32_t)((lane & 3) * rh + bn * 8 + (lane >> 2));
#pragma unroll
  for (int kk = 0; kk < RM / 4; ++kk) {
    double fa[2], fb[2];
    const int k = 4 * kk + (lane & 3);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = (bm + q) * 8 + (lane >> 2);
      const bool in = i < r && k < r;
      const double v = in ? lds64(apk32 + 8u * (uint32_t)sm.gposT[i * r + k]) : 0.0;
      fa[q] = (in && i == k) ? v + lam : v;
      fb[q] = lds64(bc + 64u * (uint32_t)q + 32u * (uint32_t)(kk * rh));
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
        sts64(o32 + 8u * (uint32_t)(i * rh + c), 2.0 * dl - acc[q][p][h]);
        if (i < r && c < r) emax = fmax(emax, fabs(dl - acc[q][p][h]));
      }
    }
  return emax;
}

// A^-1 (A = sm.Am, SPD) -> out (row stride os) by the symmetric sweep operator (Gauss-Jordan,
// one pivot per barrier; thread t owns row t/8, columns t%8 + 8u).  A zero pivot of the PSD
// matrix is a zero row/column: the min-norm (lstsq, cp.py:176-177) answer.  Returns 1 on a
// negative / non-finite pivot.  All threads.
template <int RM>
__device__ int rw_inverse(const RowsArgs& a, const RwSmem& sm, double* out, int os) {
  constexpr int EPT = RM / 8;
  const int r = a.r, rh = rw_pad4(r), t = threadIdx.x;
  const int i = t >> 3, c0 = t & 7;
  double* pub = sm.pub;
  double v[EPT];
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int c = c0 + 8 * u;
    v[u] = (i < r && c < r) ? sm.Am[i * rh + c] : 0.0;
  }
  if (i == 0)
#pragma unroll
    for (int u = 0; u < EPT; ++u) pub[c0 + 8 * u] = v[u];
  __syncthreads();
  int bad = 0;
  for (int k = 0; k < r; ++k) {
    const double* rk = pub + (k & 1) * 36;
    double* rn = pub + ((k + 1) & 1) * 36;
    const double d = rk[k];
    if (d < 0.0 || !isfinite(d)) bad = 1;
    const double id = (d == 0.0) ? 0.0 : rcp_nr(d);
    const double f = (i < r ? rk[i] : 0.0) * id;
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + 8 * u;
      const double akc = rk[c];
      double nv = fma(-f, akc, v[u]);
      nv = (c == k) ? f : nv;
      nv = (i == k) ? ((c == k) ? -id : akc * id) : nv;
      v[u] = nv;
    }
    if (i == k + 1)
#pragma unroll
      for (int u = 0; u < EPT; ++u) rn[c0 + 8 * u] = v[u];
    __syncthreads();
  }
  if (i < r)
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + 8 * u;
      if (c < r) out[i * os + c] = -v[u];
    }
  __syncthreads();
  return bad;
}

// RM x RM product P = A B (row stride rh, K = RM, zero padded), one 8x8 tile per item on
// warps [w0, w0 + nw) (DMMA, two interleaved K chains).  mode 0: out = 2I - P and returns this
// thread's max |I - P|_ic (i, c < r); mode 1: out = P.
template <int RM>
__device__ double rw_gemm(const double* A, const double* B, double* out, int rh, int r, int mode, int nw, int w0 = 0) {
  constexpr int MT = RM / 8;
  const int warp = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
  const uint32_t a32 = smem_u32(A), b32 = smem_u32(B), o32 = smem_u32(out);
  double emax = 0.0;
  if (RM == 32 && nw == 4) {
    // four warps: warp w owns the 2 x 2 block of 8 x 8 tiles (2 (w / 2) + {0, 1}, 2 (w % 2) + {0, 1});
    // four independent DMMA chains per K step, A / B fragments shared along the block
    const int bm = 2 * (warp >> 1), bn = 2 * (warp & 1);
    double acc[2][2][2] = {};
    const uint32_t ar = a32 + 8u * (uint32_t)((bm * 8 + (lane >> 2)) * rh + (lane & 3));
    const uint32_t bc = b32 + 8u * (uint32_t)((lane & 3) * rh + bn * 8 + (lane >> 2));
#pragma unroll
    for (int kk = 0; kk < RM / 4; ++kk) {
      double fa[2], fb[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        fa[q] = lds64(ar + 8u * (uint32_t)(q * 8 * rh) + 32u * (uint32_t)kk);
        fb[q] = lds64(bc + 64u * (uint32_t)q + 32u * (uint32_t)(kk * rh));
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int p = 0; p < 2; ++p) dmma_8x8x4(acc[q][p][0], acc[q][p][1], fa[q], fb[p]);
    }
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
            sts64(o32 + 8u * (uint32_t)(i * rh + c), 2.0 * dl - acc[q][p][h]);
            if (i < r && c < r) emax = fmax(emax, fabs(dl - acc[q][p][h]));
          } else {
            sts64(o32 + 8u * (uint32_t)(i * rh + c), acc[q][p][h]);
          }
        }
      }
    return emax;
  }
  for (int it = warp; it < MT * MT; it += nw) {
    const int m = it / MT, n = it - m * MT;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    const uint32_t arow = a32 + 8u * (uint32_t)((m * 8 + (lane >> 2)) * rh + (lane & 3));
    const uint32_t bcol = b32 + 8u * (uint32_t)((lane & 3) * rh + n * 8 + (lane >> 2));
#pragma unroll
    for (int kk = 0; kk < RM / 4; kk += 2) {
      const double a0 = lds64(arow + 32u * (uint32_t)kk), a1 = lds64(arow + 32u * (uint32_t)(kk + 1));
      const double b0 = lds64(bcol + 32u * (uint32_t)(kk * rh)), b1 = lds64(bcol + 32u * (uint32_t)((kk + 1) * rh));
      dmma_8x8x4(c0, c1, a0, b0);
      if (kk + 1 < RM / 4) dmma_8x8x4(c2, c3, a1, b1);
    }
    const double acc[2] = {c0 + c2, c1 + c3};
    const int i = m * 8 + (lane >> 2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = n * 8 + 2 * (lane & 3) + h;
      const double dl = (i == c) ? 1.0 : 0.0;
      if (mode == 0) {
        sts64(o32 + 8u * (uint32_t)(i * rh + c), 2.0 * dl - acc[h]);
        if (i < r && c < r) emax = fmax(emax, fabs(dl - acc[h]));
      } else {
        sts64(o32 + 8u * (uint32_t)(i * rh + c), acc[h]);
      }
    }
  }
  return emax;
}

// NS independent 8x8 DMMA chains: acc[u] += A^T B_u over ksteps x 4 rows; A rows at
// a0 + s * arow (lane column fixed), B_u rows at b[u] + s * bst[u] (32-bit shared
// addresses, no predicates: padding rows are zero, stray lanes feed discarded outputs)
template <int NS>
__device__ __forceinline__ void rw_chains(uint32_t a0, uint32_t arow, const uint32_t* b, const uint32_t* bst, int ksteps,
                                          double (&acc)[NS][2]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < NS; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll 2
  for (int kk = 0; kk < ksteps; ++kk) {
    const uint32_t s = 4u * (uint32_t)kk + (uint32_t)(lane & 3);
    const double fa = lds64(a0 + s * arow);
    double fb[NS];
#pragma unroll
    for (int u = 0; u < NS; ++u) fb[u] = lds64(b[u] + s * bst[u]);
#pragma unroll
    for (int u = 0; u < NS; ++u) dmma_8x8x4(acc[u][0], acc[u][1], fa, fb[u]);
  }
}

struct RwCtx {
  int b, c, S, P, w, c0;   // rank in cluster, cluster (slab), sizes, slab width / start
  int oc0, wc;             // owned slab columns [oc0, oc0 + wc)
  uint32_t in_bytes;       // bytes an exchange delivers into this CTA's inbox (the S - 1 peers' pieces)
  uint32_t pub_bytes;      // bytes the publishes of an exchange deliver (had rows + A blocks)
  int gcnt;                // packed Gram entries this CTA owns
};

#define RW_PROF(i)                                                   \
  do {                                                               \
    if (a.prof && (int)blockIdx.x == a.prof_cta && threadIdx.x == 0) {    \
      const long long t_ = clock64();                                \
      prof_acc[i] += t_ - prof_t;                                    \
      prof_t = t_;                                                   \
    }                                                                \
  } while (0)

// Cluster exchange for mode k (sm.Us = U_k[block rows], rows past the block zero).
//  1. partial cross C^T[c][l] = sum_s V_k[s][c] U_k[s][l] and the upper Gram tiles
//     sum_s U_k[s][l] U_k[s][m] on DMMA into local staging (C^T rows = slab columns;
//     Gram entries owner-major packed);
//  2. pushes: owner o receives, in inbox slot b, its contiguous column rows of C^T and
//     its packed Gram block (st.async: the bytes complete on the owner's inbox mbarrier);
//  3. the owner waits for its S-1 contributions, sums them in rank order, keeps C_k[:, own
//     columns], writes its columns of had_{hmode} = prod_{k' != hmode} C_k' (hmode >= 0)
//     into its had rows and its Gram block (+ the overlap partial sum_{l, own c} prod_k C_k
//     if want_ovl) into Gp[k];
//  4. publishes of those had rows / the Gram block to every peer (st.async onto the peers'
//     publish mbarriers); wait for the peers' publishes.
// No cluster barrier: every buffer is rewritten only after its reader's own later stores
// were received (push m+1 needs publish m, publish m+1 needs push m+1).
template <int RM>
__device__ void rw_exchange(const RowsArgs& a, const RwSmem& sm, const RwCtx& x, int k, int hmode, bool want_ovl,
                            uint32_t& ph_in, uint32_t& ph_pub, long long* prof_acc, long long& prof_t) {
  constexpr int MT = RM / 8;
  const int r = a.r, rh = rw_pad4(r), rs2 = a.rs2, wcol = a.wcol, piece = a.piece, S = x.S, gs = a.gstride;
  const int ng = r * (r + 1) / 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nb = sm.nbT[k], ksteps = (nb + 3) / 4;
  const int ntc = (x.w + 7) / 8, ncg = (ntc + 1) / 2, ngt = MT * (MT + 1) / 2;   // C items: 2 column tiles
  const int nci = MT * ncg, nitems = nci + ngt;
  double* cst = sm.scr;                  // [w][rs2] partial staging
  double* gst = sm.scr + a.cst_len;      // [S][gs]
  const uint32_t cst32 = smem_u32(cst), gst32 = smem_u32(gst);
  const uint32_t us32 = smem_u32(sm.Us), vs32 = smem_u32(sm.Vs + (size_t)a.vrow[k] * a.ldw);
  if (tid == 0) {   // this phase's expected bytes (peers may already be sending: tx count goes negative)
    mbar_arrive_expect_tx(sm.bar + 1, x.in_bytes);
    mbar_arrive_expect_tx(sm.bar + 2, hmode >= 0 ? x.pub_bytes : 0u);
  }
  // ---- 1. partials into local staging
  for (int it = warp; it < nitems; it += RW_NW) {
    if (it < nci) {
      const int m = it / MT, n = it - m * MT;   // m: pair of slab-column tiles, n: l tile
      uint32_t bb[2], bst[2];
      const uint32_t a_l = us32 + 8u * (uint32_t)(n * 8 + (lane >> 2));
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        int ct = 2 * m + u;
        if (ct >= ntc) ct = ntc - 1;
        bb[u] = vs32 + 8u * (uint32_t)(ct * 8 + (lane >> 2));
        bst[u] = 8u * (uint32_t)a.ldw;
      }
      double acc[2][2];
      rw_chains<2>(a_l, 8u * (uint32_t)rh, bb, bst, ksteps, acc);
      const int l = n * 8 + (lane >> 2);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ct = 2 * m + u;
        if (ct >= ntc || l >= r) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = ct * 8 + 2 * (lane & 3) + h;
          if (c < x.w) sts64(cst32 + 8u * (uint32_t)(c * rs2 + l), acc[u][h]);
        }
      }
    } else {
      int g = it - nci, ti = 0;
      while (g >= MT - ti) { g -= MT - ti; ++ti; }
      const int tj = ti + g;
      const uint32_t bb[1] = {us32 + 8u * (uint32_t)(tj * 8 + (lane >> 2))}, bst[1] = {8u * (uint32_t)rh};
      double acc[1][2];
      rw_chains<1>(us32 + 8u * (uint32_t)(ti * 8 + (lane >> 2)), 8u * (uint32_t)rh, bb, bst, ksteps, acc);
      const int i = ti * 8 + (lane >> 2);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tj * 8 + 2 * (lane & 3) + h;
        if (i < r && c < r && i <= c) sts64(gst32 + 8u * (uint32_t)sm.gposT[i * r + c], acc[0][h]);
      }
    }
  }
  __syncthreads();
  RW_PROF(14);
  // ---- 2. pushes: owner q <- (C^T rows [oc0(q), oc1(q)), Gram block q) into its slot b
  {
    const uint32_t slot = smem_u32(sm.inbox) + 8u * (uint32_t)(x.b * piece);
    const uint32_t bar_in = smem_u32(sm.bar + 1);
    for (int q = warp; q < S; q += RW_NW) {
      if (q == x.b) continue;
      const int q0 = sm.ocT[q], nq = sm.ocT[q + 1] - q0;
      const int nc2 = nq * rs2 / 2;
      const uint32_t dst = mapa_u32(slot, (uint32_t)q), rbar = mapa_u32(bar_in, (uint32_t)q);
      const uint32_t src = cst32 + 8u * (uint32_t)(q0 * rs2);
      for (int e = lane; e < nc2; e += 32) {
        const double2 v = lds2x64(src + 16u * (uint32_t)e);
        st_async_v2(dst + 16u * (uint32_t)e, v.x, v.y, rbar);
      }
      const uint32_t gsrc = gst32 + 8u * (uint32_t)(q * gs);
      const uint32_t gdst = dst + 8u * (uint32_t)(wcol * rs2);
      for (int e = lane; e < gs / 2; e += 32) {
        const double2 v = lds2x64(gsrc + 16u * (uint32_t)e);
        st_async_v2(gdst + 16u * (uint32_t)e, v.x, v.y, rbar);
      }
    }
  }
  RW_PROF(9);
  mbar_wait(sm.bar + 1, ph_in);
  ph_in ^= 1u;
  RW_PROF(10);
  // ---- 3. owner: fixed-order sums (rank order; own contribution from the staging)
  double* Ck = sm.Cown + (size_t)k * wcol * r;
  const int ncr = x.wc * r, nred = ncr + gs;
  for (int e = tid; e < nred; e += RW_NT) {
    const bool isc = e < ncr;
    int own, ii;
    if (isc) {
      const int dv = sm.divT[e], cc = dv & 0xffff, l = dv >> 16;
      ii = cc * rs2 + l;
      own = (x.oc0 + cc) * rs2 + l;
    } else {
      ii = wcol * rs2 + (e - ncr);
      own = a.cst_len + x.b * gs + (e - ncr);
    }
    // all S contributions issued together through 32-bit shared addresses, summed in rank order
    const uint32_t ib = smem_u32(sm.inbox) + 8u * (uint32_t)ii, pst = 8u * (uint32_t)piece;
    const double ownv = lds64(cst32 + 8u * (uint32_t)own);
    double pv[16];
#pragma unroll
    for (int src = 0; src < 16; ++src) pv[src] = src < S ? lds64(ib + (uint32_t)src * pst) : 0.0;
    double v = 0.0;
#pragma unroll
    for (int src = 0; src < 16; ++src) v += (src == x.b) ? ownv : pv[src];
    if (isc) Ck[e] = v;
    else sm.gpub[e - ncr] = v;
  }
  __syncthreads();
  RW_PROF(12);
  // this rank's Gram block of mode k stays local; with hmode >= 0 it publishes its block of
  // A_hmode = prod_{k' != hmode} G_k' (+ the overlap / self-Gram partials of the residual)
  double* Ab = sm.Apk + (size_t)x.b * gs;
  // multicast staging of this exchange (double-buffered by exchange parity)
  double* Hgc = a.mc ? a.Hg + ((size_t)ph_pub * x.P + x.c) * (size_t)a.kpad * rh : nullptr;
  double* Agc = a.mc ? a.Ag + ((size_t)ph_pub * x.P + x.c) * (size_t)S * gs : nullptr;
  const int gcnt = x.gcnt;
  for (int e = tid; e < gs; e += RW_NT) sm.Gown[(size_t)k * gs + e] = sm.gpub[e];
  if (want_ovl) {
    double ovl = 0.0, self = 0.0;
    for (int e = tid; e < ncr; e += RW_NT) {
      double v = 1.0;
      for (int kk = 0; kk < a.d; ++kk) v *= sm.Cown[(size_t)kk * wcol * r + e];
      ovl += v;
    }
    for (int e = tid; e < gcnt; e += RW_NT) {
      double v = sm.gpub[e];
      for (int kk = 0; kk < a.d; ++kk)
        if (kk != k) v *= sm.Gown[(size_t)kk * gs + e];
      self += sm.gdiag[e] ? v : 2.0 * v;
    }
    ovl = rw_block_sum(ovl, sm.part);
    self = rw_block_sum(self, sm.part);
    if (tid == 0) {
      Ab[gs - 1] = ovl; Ab[gs - 2] = self;
      if (a.mc) { Agc[(size_t)x.b * gs + gs - 1] = ovl; Agc[(size_t)x.b * gs + gs - 2] = self; }
    }
  }
  if (hmode >= 0) {
    // (32-bit shared addresses: one IMAD per operand instead of 64-bit generic address math)
    const uint32_t gown32 = smem_u32(sm.Gown), cown32 = smem_u32(sm.Cown);
    const uint32_t gstep = 8u * (uint32_t)gs, cstep = 8u * (uint32_t)(wcol * r);
    for (int e = tid; e < gs - 2; e += RW_NT) {
      double v = 0.0;
      if (e < gcnt) {
        double f[TP_MAXD];
#pragma unroll
        for (int kk = 0; kk < TP_MAXD; ++kk)
          f[kk] = (kk < a.d && kk != hmode)
                      ? (kk == k ? sm.gpub[e] : lds64(gown32 + (uint32_t)kk * gstep + 8u * (uint32_t)e))
                      : 1.0;
        v = 1.0;
#pragma unroll
        for (int kk = 0; kk < TP_MAXD; ++kk) v *= f[kk];
      }
      Ab[e] = v;
      if (a.mc) Agc[(size_t)x.b * gs + e] = v;
    }
    RW_PROF(15);
    for (int e = tid; e < ncr; e += RW_NT) {
      const int dv = sm.divT[e], cc = dv & 0xffff, l = dv >> 16;
      double f[TP_MAXD];
#pragma unroll
      for (int kk = 0; kk < TP_MAXD; ++kk)
        f[kk] = (kk < a.d && kk != hmode) ? lds64(cown32 + (uint32_t)kk * cstep + 8u * (uint32_t)e) : 1.0;
      double v = 1.0;
#pragma unroll
      for (int kk = 0; kk < TP_MAXD; ++kk) v *= f[kk];
      if (a.mc) Hgc[(size_t)(x.oc0 + cc) * rh + l] = v;
      else sm.hadT[(size_t)(x.oc0 + cc) * rh + l] = v;
    }
    if (a.mc)   // zero row padding (multicast whole rows)
      for (int cc = tid; cc < x.wc; cc += RW_NT)
        for (int l = r; l < rh; ++l) Hgc[(size_t)(x.oc0 + cc) * rh + l] = 0.0;
  }
  __syncthreads();
  RW_PROF(13);
  // ---- 4. publish the had rows and the Gram block to every peer
  if (a.mc) {
    // one TMA multicast per block: read once from L2, delivered into every CTA's had rows /
    // A block (same offsets), completing on each CTA's publish mbarrier
    if (hmode >= 0 && tid == 0) {
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      const uint16_t mask = (uint16_t)((1u << S) - 1u);
      const uint32_t bar_pub = smem_u32(sm.bar + 2);
      if (x.wc > 0)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
            "[%3], %4;\n" ::"r"(smem_u32(sm.hadT) + 8u * (uint32_t)(x.oc0 * rh)),
            "l"(Hgc + (size_t)x.oc0 * rh), "r"((uint32_t)(x.wc * rh * 8)), "r"(bar_pub), "h"(mask)
            : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
          "[%3], %4;\n" ::"r"(smem_u32(Ab)),
          "l"(Agc + (size_t)x.b * gs), "r"((uint32_t)(gs * 8)), "r"(bar_pub), "h"(mask)
          : "memory");
    }
  } else {
    const uint32_t hsrc = smem_u32(sm.hadT) + 8u * (uint32_t)(x.oc0 * rh);
    const uint32_t gsrc = smem_u32(Ab);
    const uint32_t bar_pub = smem_u32(sm.bar + 2);
    const int nh2 = hmode >= 0 ? x.wc * (r / 2) : 0;
    for (int q = warp; q < S && hmode >= 0; q += RW_NW) {
      if (q == x.b) continue;
      const uint32_t rbar = mapa_u32(bar_pub, (uint32_t)q), hdst = mapa_u32(hsrc, (uint32_t)q);
      if (!(r & 1)) {
        for (int e = lane; e < nh2; e += 32) {
          const int dv = sm.divT[2 * e], cc = dv & 0xffff, l = dv >> 16;   // (r even: l even)
          const double2 v = *reinterpret_cast<const double2*>(sm.hadT + (size_t)(x.oc0 + cc) * rh + l);
          st_async_v2(hdst + 8u * (uint32_t)(cc * rh + l), v.x, v.y, rbar);
        }
      } else if (hmode >= 0) {
        for (int e = lane; e < x.wc * r; e += 32) {
          const int dv = sm.divT[e], cc = dv & 0xffff, l = dv >> 16;
          st_async_f64(hdst + 8u * (uint32_t)(cc * rh + l), sm.hadT[(size_t)(x.oc0 + cc) * rh + l], rbar);
        }
      }
      const uint32_t gdst = mapa_u32(gsrc, (uint32_t)q);
      for (int e = lane; e < gs / 2; e += 32) {
        const double2 v = *reinterpret_cast<const double2*>(Ab + 2 * e);
        st_async_v2(gdst + 16u * (uint32_t)e, v.x, v.y, rbar);
      }
    }
  }
  RW_PROF(11);
  mbar_wait(sm.bar + 2, ph_pub);
  ph_pub ^= 1u;
}

// cross-cluster round u: release this CTA's slot flag / acquire the P flags of row block b
__device__ __forceinline__ void rw_flag(const RowsArgs& a, const RwCtx& x, int u) {
  unsigned int* f = a.flags + ((size_t)(u & 1) * x.S + x.b) * x.P + x.c;
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(f), "r"((unsigned int)(u + 1)) : "memory");
}

__device__ __forceinline__ void rw_wait(const RowsArgs& a, const RwCtx& x, int u, int& status) {
  if (threadIdx.x < x.P && !(status & 4)) {
    const unsigned int* f = a.flags + ((size_t)(u & 1) * x.S + x.b) * x.P + threadIdx.x;
    const unsigned int want = (unsigned int)(u + 1);
    const long long t0 = clock64();
    unsigned int v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
      if ((int)(v - want) >= 0) break;
      if (clock64() - t0 > 8000000000LL) { status |= 4; break; }   // ~4 s: a missing peer
    }
  }
  if (__syncthreads_or(status & 4)) status |= 4;
}

template <int RM>
__global__ void __launch_bounds__(RW_NT, 1) als_rows(const __grid_constant__ RowsArgs a) {
  extern __shared__ __align__(16) double smem[];
  constexpr int NT = RM / 8;
  if (a.run_if && *a.run_if == 0) return;   // (uniform: the fallback launch behind the Gram-space kernel)
  const RwSmem sm = rw_carve(smem, a, RM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  long long prof_t = clock64(), prof_acc[16] = {};
  RwCtx x;
  x.S = a.S; x.P = a.P;
  x.b = (int)cluster_rank();
  x.c = blockIdx.x / a.S;
  x.c0 = (int)((long long)a.R * x.c / a.P);
  x.w = (int)((long long)a.R * (x.c + 1) / a.P) - x.c0;
  x.oc0 = x.w * x.b / a.S; x.wc = x.w * (x.b + 1) / a.S - x.oc0;
  const int r = a.r, rh = rw_pad4(r), d = a.d, ldw = a.ldw;
  const size_t xsz = (size_t)RM * rh;
  double* Xw = a.Xw + (size_t)blockIdx.x * d * xsz;   // this CTA's warm starts (one per mode)
  int status = 0;

  // ---- setup: zero everything (padding rows / columns stay zero), V blocks, initial crosses
  {
    const size_t tot = rw_smem_doubles(a, RM);
    for (size_t e = tid; e < tot; e += RW_NT) smem[e] = 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) mbar_init(sm.bar + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const int ng = r * (r + 1) / 2;
    for (int e = tid; e < r * r; e += RW_NT) {
      int i = e / r, c = e - (e / r) * r;
      if (i > c) { const int t = i; i = c; c = t; }
      const int p = i * r - (i * (i - 1)) / 2 + (c - i), o = (a.S * (p + 1) - 1) / ng;
      sm.gposT[e] = o * a.gstride + p - (ng * o) / a.S;
    }
    for (int e = tid; e < rw_tbl(a); e += RW_NT) sm.divT[e] = (e / r) | ((e % r) << 16);
    for (int k = tid; k < d; k += RW_NT) {
      sm.qb0T[k] = a.q[k] * x.b / a.S;
      sm.nbT[k] = a.q[k] * (x.b + 1) / a.S - sm.qb0T[k];
    }
    for (int q = tid; q <= a.S; q += RW_NT) sm.ocT[q] = x.w * q / a.S;
    for (int e = tid; e < a.gstride; e += RW_NT) sm.gdiag[e] = 0;
    __syncthreads();
    for (int i = tid; i < r; i += RW_NT) {
      const int pos = sm.gposT[i * r + i];
      if (pos / a.gstride == x.b) sm.gdiag[pos - x.b * a.gstride] = 1;
    }
  }
  __syncthreads();
  {
    const int gs = a.gstride;
    uint32_t pub = 0;
    for (int q = 0; q < a.S; ++q) {
      if (a.mc) pub += (uint32_t)(((sm.ocT[q + 1] - sm.ocT[q]) * rh + gs) * 8);   // every owner, self incl.
      else if (q != x.b) pub += (uint32_t)(((sm.ocT[q + 1] - sm.ocT[q]) * r + gs) * 8);
    }
    x.pub_bytes = pub;
    x.in_bytes = (uint32_t)((a.S - 1) * (x.wc * a.rs2 + gs) * 8);
    const int ng = r * (r + 1) / 2;
    x.gcnt = (ng * (x.b + 1)) / a.S - (ng * x.b) / a.S;
  }
  for (int k = 0; k < d; ++k) {
    const int qb0 = sm.qb0T[k], nb = sm.nbT[k];
    const double* Vk = a.V + a.offV[k] + (size_t)qb0 * a.R + x.c0;
    double* vs = sm.Vs + (size_t)a.vrow[k] * ldw;
    for (int e = tid; e < nb * x.w; e += RW_NT) {
      const int s = e / x.w, cc = e - s * x.w;
      vs[s * ldw + cc] = __ldg(Vk + (size_t)s * a.R + cc);
    }
  }
  cluster_barrier();   // every CTA of the cluster is running and zeroed before remote stores
  uint32_t ph_in = 0, ph_pub = 0;
  for (int k = 0; k < d; ++k) {
    const int qb0 = sm.qb0T[k], nb = sm.nbT[k];
    const double* Uk = a.U + a.offU[k] + (size_t)qb0 * r;
    for (int e = tid; e < rw_nbr(a) * rh; e += RW_NT) {
      const int s = e / rh, l = e - s * rh;
      sm.Us[e] = (s < nb && l < r) ? __ldcg(Uk + (size_t)s * r + l) : 0.0;
    }
    __syncthreads();
    rw_exchange<RM>(a, sm, x, k, k == d - 1 ? 0 : -1, false, ph_in, ph_pub, prof_acc, prof_t);
  }

  const double norm_sq = a.need_resid ? fmax(*a.norm_sq, 0.0) : 0.0;
  const double t_norm = sqrt(norm_sq);
  double prev = INFINITY;
  int u = 0, done = 0;
  uint32_t xph = 0;
  const int nwrite = x.c == 0;   // cluster 0 writes the iterate (all clusters hold it)
  const size_t slot_stride = (size_t)a.ylen;
  for (int sweep = 0; sweep < a.sweeps; ++sweep) {
    for (int j = 0; j < d; ++j) {
      RW_PROF(0);
      const bool warm = sweep > 0 && a.ns;
      if (warm && tid == 0) {   // this mode's warm start (written by this CTA one sweep ago)
        fence_proxy_async();
        mbar_arrive_expect_tx(sm.bar, (uint32_t)(xsz * 8));
        bulk_g2s(sm.X0, Xw + (size_t)j * xsz, (uint32_t)(xsz * 8), sm.bar);
      }
      const int nb = sm.nbT[j], qb0 = sm.qb0T[j], mtr = (nb + 7) / 8;
      double* slot = a.Y + (((size_t)(u & 1) * x.S + x.b) * x.P + x.c) * slot_stride;
      bool ok = false;
      if (a.split) {
        // ---- 1'. warps 0-3: partial rhs Y = V_j[blk, slab] had^T straight to the slot, then
        // warp 0 releases it; warps 4-7 at the same time: A_j and the warm-started inverse
        // (both only need the previous exchange's publishes)
        if (warp < 4) {
          // warp w owns column tile n = w (+4 ...) and walks the row tiles in pairs: the had
          // fragment is shared by both row tiles, two K chains each -> four independent chains
          const int kst = (x.w + 3) / 4;
          const uint32_t vs32 = smem_u32(sm.Vs + (size_t)a.vrow[j] * ldw), hd32 = smem_u32(sm.hadT);
          for (int n = warp; n < NT; n += 4) {
            const uint32_t brow = hd32 + 8u * (uint32_t)((lane & 3) * rh + n * 8 + (lane >> 2));
            for (int m0 = 0; m0 < mtr; m0 += 2) {
              const bool two = m0 + 1 < mtr;   // (warp-uniform)
              const uint32_t ar0 = vs32 + 8u * (uint32_t)((m0 * 8 + (lane >> 2)) * ldw + (lane & 3));
              const uint32_t ar1 = ar0 + 64u * (uint32_t)ldw;
              double c[2][2][2] = {};   // [row tile][chain][half]
              int kk = 0;
              for (; kk + 1 < kst; kk += 2) {
                const double b0 = lds64(brow + 32u * (uint32_t)(kk * rh)), b1 = lds64(brow + 32u * (uint32_t)((kk + 1) * rh));
                const double a00 = lds64(ar0 + 32u * (uint32_t)kk), a01 = lds64(ar0 + 32u * (uint32_t)(kk + 1));
                dmma_8x8x4(c[0][0][0], c[0][0][1], a00, b0);
                dmma_8x8x4(c[0][1][0], c[0][1][1], a01, b1);
                if (two) {
                  const double a10 = lds64(ar1 + 32u * (uint32_t)kk), a11 = lds64(ar1 + 32u * (uint32_t)(kk + 1));
                  dmma_8x8x4(c[1][0][0], c[1][0][1], a10, b0);
                  dmma_8x8x4(c[1][1][0], c[1][1][1], a11, b1);
                }
              }
              if (kk < kst) {
                const double b0 = lds64(brow + 32u * (uint32_t)(kk * rh)), a00 = lds64(ar0 + 32u * (uint32_t)kk);
                dmma_8x8x4(c[0][0][0], c[0][0][1], a00, b0);
                if (two) {
                  const double a10 = lds64(ar1 + 32u * (uint32_t)kk);
                  dmma_8x8x4(c[1][0][0], c[1][0][1], a10, b0);
                }
              }
              const int l = n * 8 + 2 * (lane & 3);
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int s = (m0 + q) * 8 + (lane >> 2);
                const double v0 = c[q][0][0] + c[q][1][0], v1 = c[q][0][1] + c[q][1][1];
                if ((q == 0 || two) && s < nb && l < r) {
                  if (l + 1 < r && !(r & 1)) *reinterpret_cast<double2*>(slot + s * r + l) = make_double2(v0, v1);
                  else { slot[s * r + l] = v0; if (l + 1 < r) slot[s * r + l + 1] = v1; }
                }
              }
            }
          }
          bar_named(2, 128);   // every slot store of the group issued
          RW_PROF(7);
          if (tid == 0) rw_flag(a, x, u);
        } else if (warm) {
          double em;
          if (RM == 32) {   // A_j read from the packed blocks (no unpack on this path)
            const double lam = rw_lambda(a, sm);
            mbar_wait(sm.bar, xph);
            em = rw_ns_packed(a, sm, lam, sm.X0, sm.scr, 4);                 // T = 2I - A X0, |I - A X0|
          } else {
            rw_build_a_w(a, sm, 128, 128);
            mbar_wait(sm.bar, xph);
            em = rw_gemm<RM>(sm.Am, sm.X0, sm.scr, rh, r, 0, 4, 4);
          }
          {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
            if (lane == 0) sm.part[warp - 4] = em;
            bar_named(1, 128);
            rw_gemm<RM>(sm.X0, sm.scr, sm.X1, rh, r, 1, 4, 4);                // X1 = X0 T
          }
        }
        if (warm) xph ^= 1u;
        __syncthreads();
        if (warm) {
          double em = 0.0;
          for (int q = 0; q < 4; ++q) em = fmax(em, sm.part[q]);
          ok = em <= 1e-8;   // (NaN fails)
        }
        if (!ok) rw_build_a_w(a, sm, RW_NT);   // the exact sweep below reads the unpacked A_j
      } else {
        // ---- 1. partial rhs Y = V_j[blk, slab] had^T (M = s, N = l, K = c) straight to the slot
        {
          const int kst = (x.w + 3) / 4;
          int kparts = 1;
          while (mtr * NT * kparts * 2 <= RW_NW) kparts *= 2;
          const int per = (kst + kparts - 1) / kparts, items = mtr * NT * kparts;
          const uint32_t vs32 = smem_u32(sm.Vs + (size_t)a.vrow[j] * ldw), hd32 = smem_u32(sm.hadT);
          for (int it = warp; it < items; it += RW_NW) {
            const int mn = it / kparts, kp = it - mn * kparts, m = mn / NT, n = mn - m * NT;
            const int kb = kp * per, ke = min(kst, kb + per);
            const int s = m * 8 + (lane >> 2);
            const uint32_t arow = vs32 + 8u * (uint32_t)(s * ldw + (lane & 3));
            const uint32_t brow = hd32 + 8u * (uint32_t)((lane & 3) * rh + n * 8 + (lane >> 2));
            double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
            int kk = kb;
            for (; kk + 1 < ke; kk += 2) {   // two independent chains
              const double a0 = lds64(arow + 32u * (uint32_t)kk), a1 = lds64(arow + 32u * (uint32_t)(kk + 1));
              const double b0 = lds64(brow + 8u * (uint32_t)(4 * kk * rh)), b1 = lds64(brow + 8u * (uint32_t)(4 * (kk + 1) * rh));
              dmma_8x8x4(acc0, acc1, a0, b0);
              dmma_8x8x4(acc2, acc3, a1, b1);
            }
            if (kk < ke) {
              const double a0 = lds64(arow + 32u * (uint32_t)kk), b0 = lds64(brow + 8u * (uint32_t)(4 * kk * rh));
              dmma_8x8x4(acc0, acc1, a0, b0);
            }
            acc0 += acc2;
            acc1 += acc3;
            if (kparts == 1) {
              const int l = n * 8 + 2 * (lane & 3);
              if (s < nb && l < r) {
                if (l + 1 < r && !(r & 1)) *reinterpret_cast<double2*>(slot + s * r + l) = make_double2(acc0, acc1);
                else { slot[s * r + l] = acc0; if (l + 1 < r) slot[s * r + l + 1] = acc1; }
              }
            } else {
              sm.scr[(size_t)it * 64 + 2 * lane] = acc0;
              sm.scr[(size_t)it * 64 + 2 * lane + 1] = acc1;
            }
          }
          if (kparts > 1) {
            __syncthreads();
            for (int e = tid; e < nb * r; e += RW_NT) {
              const int s = e / r, l = e - s * r, m = s >> 3, n = l >> 3;
              const int ln = ((s & 7) << 2) | ((l & 7) >> 1), h = l & 1;
              double v = 0.0;
              for (int kp = 0; kp < kparts; ++kp) v += sm.scr[((size_t)(m * NT + n) * kparts + kp) * 64 + 2 * ln + h];
              slot[e] = v;
            }
          }
        }
        RW_PROF(7);
        // ---- A_j and its inverse while the peers' slots land: the last warp releases this
        // CTA's slot (the gpu-scope release drains the stores) while the others build A_j and
        // refine the warm start
        __syncthreads();   // every slot store issued
        RW_PROF(8);
        {
          constexpr int NWK = RW_NW - 1;
          if (warp == RW_NW - 1) {
            if (lane == 0) rw_flag(a, x, u);
          } else {
            rw_build_a_w(a, sm, NWK * 32);
            if (warm) {
              mbar_wait(sm.bar, xph);
              double em = rw_gemm<RM>(sm.Am, sm.X0, sm.scr, rh, r, 0, NWK);   // T = 2I - A X0, |I - A X0|
  #pragma unroll
              for (int o = 16; o > 0; o >>= 1) em = fmax(em, __shfl_xor_sync(0xffffffffu, em, o));
              if (lane == 0) sm.part[warp] = em;
              bar_named(1, NWK * 32);
              rw_gemm<RM>(sm.X0, sm.scr, sm.X1, rh, r, 1, NWK);                // X1 = X0 T
            }
          }
          if (warm) xph ^= 1u;
          __syncthreads();
          if (warm) {
            double em = 0.0;
            for (int q = 0; q < NWK; ++q) em = fmax(em, sm.part[q]);
            // one step squares the error: |I - A X1| <= |I - A X0|^2 <= (r * 1e-8)^2 ~ 1e-13
            ok = em <= 1e-8;   // (NaN fails)
          }
        }
      }
      RW_PROF(1);
      if (!ok) status |= rw_inverse<RM>(a, sm, sm.X1, rh);
      RW_PROF(2);
      // ---- 2. rhs = sum over the P clusters (fixed order): warp c waits for cluster c's
      // flag and stages its slot (overlapping the later flags), then the ordered sum
      {
        const int nslot = (int)rw_ev((size_t)rw_nbr(a) * r), n2 = nb * r / 2;
        const double* ybase = a.Y + (((size_t)(u & 1) * x.S + x.b) * x.P) * slot_stride;
        int bad = 0;
        // next sweep's warm start for this mode (read back only by this CTA) by the last
        // warp, while the others wait for the flags (P <= 7: the last warp polls none)
        if (a.ns && warp == RW_NW - 1)
          for (int e = lane; e < (int)xsz; e += 32) Xw[(size_t)j * xsz + e] = sm.X1[e];
        for (int cc = warp; cc < x.P; cc += RW_NW) {
          if (lane == 0 && !(status & 4)) {
            const unsigned int* f = a.flags + ((size_t)(u & 1) * x.S + x.b) * x.P + cc;
            const unsigned int want = (unsigned int)(u + 1);
            const long long t0 = clock64();
            unsigned int v;
            for (;;) {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
              if ((int)(v - want) >= 0) break;
              if (clock64() - t0 > 8000000000LL) { bad = 4; break; }   // ~4 s: a missing peer
            }
          }
          __syncwarp();
          const double2* src = reinterpret_cast<const double2*>(ybase + (size_t)cc * slot_stride);
          double2* dst = reinterpret_cast<double2*>(sm.scr + (size_t)cc * nslot);
          for (int e = lane; e < n2; e += 32) dst[e] = __ldcg(src + e);
          if ((nb * r) & 1)
            if (lane == 0) sm.scr[(size_t)cc * nslot + nb * r - 1] = __ldcg(ybase + (size_t)cc * slot_stride + nb * r - 1);
        }
        if (__syncthreads_or(bad)) status |= 4;
        RW_PROF(3);
        for (int e = tid; e < nb * r; e += RW_NT) {
          const int dv = sm.divT[e], sr = dv & 0xffff, l = dv >> 16;
          const uint32_t y32 = smem_u32(sm.scr) + 8u * (uint32_t)e, ystep = 8u * (uint32_t)nslot;
          double yv[RW_PMAX];
#pragma unroll
          for (int cc = 0; cc < RW_PMAX; ++cc) yv[cc] = cc < x.P ? lds64(y32 + (uint32_t)cc * ystep) : 0.0;
          double v = 0.0;
#pragma unroll
          for (int cc = 0; cc < RW_PMAX; ++cc) v += yv[cc];
          sts64(smem_u32(sm.rb) + 8u * (uint32_t)(sr * rh + l), v);
        }
      }
      __syncthreads();
      RW_PROF(4);
      {
        const uint32_t rb32 = smem_u32(sm.rb), xi32 = smem_u32(sm.X1);
        const int kst = (r + 3) / 4, items = mtr * NT;
        int nf = 0;
        for (int it = warp; it < items; it += RW_NW) {
          const int m = it / NT, n = it - m * NT;
          const int s = m * 8 + (lane >> 2);
          double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
          for (int kk = 0; kk < kst; ++kk) {
            const uint32_t kr = 4u * (uint32_t)kk + (uint32_t)(lane & 3);
            const double fa = lds64(rb32 + 8u * (uint32_t)(s * rh) + 8u * kr);
            const double fb = lds64(xi32 + 8u * (kr * (uint32_t)rh + (uint32_t)(n * 8 + (lane >> 2))));
            dmma_8x8x4(acc0, acc1, fa, fb);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = n * 8 + 2 * (lane & 3) + h;
            const double v = h ? acc1 : acc0;
            const uint32_t ua = smem_u32(sm.Us) + 8u * (uint32_t)(s * rh + i);
            if (s >= nb && i < r && s < rw_nbr(a)) sts64(ua, 0.0);   // K padding of the next partials
            if (s < nb && i < r) {
              sts64(ua, v);
              if (!isfinite(v)) nf = 1;
              if (nwrite) a.U[a.offU[j] + (size_t)(qb0 + s) * r + i] = v;
            }
          }
        }
        if (nf) atomicOr(a.info, 2);
      }
      ++u;
      __syncthreads();
      RW_PROF(5);
      // ---- 3. C_j, G_j and had_{j+1} through the cluster (not after the last solve
      // unless the residual needs the final crosses)
      if (a.need_resid || sweep + 1 < a.sweeps || j + 1 < d)
        rw_exchange<RM>(a, sm, x, j, (j + 1) % d, a.need_resid && j == d - 1, ph_in, ph_pub, prof_acc, prof_t);
      RW_PROF(6);
    }
    done = sweep + 1;
    if (a.need_resid) {
      // overlap / self-Gram sums: the owners' partials in rank order, the overlap then over
      // the P clusters
      double ovc = 0.0, self = 0.0;
      for (int q = 0; q < x.S; ++q) {
        ovc += sm.Apk[(size_t)q * a.gstride + a.gstride - 1];
        self += sm.Apk[(size_t)q * a.gstride + a.gstride - 2];
      }
      double* slot = a.Y + (((size_t)(u & 1) * x.S + x.b) * x.P + x.c) * slot_stride;
      if (tid == 0) slot[a.ylen - 1] = ovc;
      __syncthreads();
      if (tid == 0) rw_flag(a, x, u);
      rw_wait(a, x, u, status);
      double ovt = 0.0;
      const double* y0 = a.Y + (((size_t)(u & 1) * x.S + x.b) * x.P) * slot_stride + (a.ylen - 1);
      for (int cc = 0; cc < x.P; ++cc) ovt += __ldcg(y0 + (size_t)cc * slot_stride);
      ++u;
      const double resid = sqrt(fmax(norm_sq - 2.0 * ovt + self, 0.0));
      if (blockIdx.x == 0 && tid == 0 && a.trace) a.trace[sweep] = resid;
      if (resid <= a.tol * t_norm) break;
      if (prev - resid < a.stall * fmax(t_norm, 1.0)) break;
      prev = resid;
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (status & 1) atomicOr(a.info, 1);
    if (status & 4) atomicOr(a.info, 4);
    a.info[1] = done;
  } else if ((status & 4) && tid == 0) {
    atomicOr(a.info, 4);
  }
  if (a.prof && (int)blockIdx.x == a.prof_cta && tid == 0)
    for (int q = 0; q < 16; ++q) a.prof[q] += prof_acc[q];
  cluster_barrier();   // no CTA exits while a peer may still store into its shared memory
}

static int g_rows_mc = 1;   // debug hook: 0 = publishes by st.async remote stores
static int g_rows_split = 1;   // debug hook: 0 = rhs product on all warps, then A_j / inverse on seven

static const void* rows_kernel(int rm) {
  switch (rm) {
    case 8: return (const void*)als_rows<8>;
    case 16: return (const void*)als_rows<16>;
    default: return (const void*)als_rows<32>;
  }
}

// P clusters of S CTAs for (d, q, R, r): fills pl.a's shape fields and the smem size.
static bool rows_try(int d, const int* q, int R, int r, int S, int P, int smem_optin, RowsPlan& pl) {
  RowsArgs& a = pl.a;
  memset(&a, 0, sizeof(a));
  a.d = d; a.R = R; a.r = r; a.S = S; a.P = P;
  const int rh = rw_pad4(r);
  a.wmax = (R + P - 1) / P;
  const int wp8 = (a.wmax + 7) / 8 * 8;
  a.ldw = rw_pad4(wp8);
  a.kpad = wp8;
  a.wcol = (a.wmax + S - 1) / S;
  a.rs2 = r + 2 - (r & 1);                        // even row stride of the C^T staging
  const int ng = r * (r + 1) / 2;
  a.gstride = (ng + S - 1) / S + 2;               // owner block of the packed Gram + overlap / self slots
  a.gstride += a.gstride & 1;
  a.piece = a.wcol * a.rs2 + a.gstride;
  a.cst_len = wp8 * a.rs2;   // (even)
  int nbmax = 0, vrow = 0;
  long long ov = 0, ou = 0;
  for (int k = 0; k < d; ++k) {
    a.q[k] = q[k];
    const int nb = (q[k] + S - 1) / S, nb4 = (nb + 3) & ~3;
    nbmax = nb4 > nbmax ? nb4 : nbmax;
    a.vrow[k] = vrow;
    vrow += nb4;
    a.offV[k] = ov; a.offU[k] = ou;
    ov += (long long)q[k] * R; ou += (long long)q[k] * r;
  }
  a.nb4max = nbmax;
  a.vtot = vrow * a.ldw;   // (8-row M tiles past the last block read the had rows that follow)
  a.ylen = nbmax * r + 2;
  a.ylen += a.ylen & 1;
  (void)rh;
  pl.smem = rw_smem_doubles(a, pl.rm) * sizeof(double);
  return pl.smem <= (size_t)smem_optin;
}

int als_rows_plan(int d, const int* q, int R, int r, int S_force, int P_force, RowsPlan& pl) {
  if (d < 2 || d > TP_MAXD || r < 1 || r > 32 || R < 1) return TP_EUNSUPPORTED;
  pl.rm = r <= 8 ? 8 : (r <= 16 ? 16 : 32);
  int dev = 0, nsm = 148, smem_optin = 227 * 1024;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  } else {
    cudaGetLastError();
  }
  int qmin = q[0];
  for (int k = 0; k < d; ++k) qmin = q[k] < qmin ? q[k] : qmin;
  const void* fn = rows_kernel(pl.rm);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  const int sizes[2] = {16, 8};
  for (int t = 0; t < 2; ++t) {
    const int S = S_force > 0 ? S_force : sizes[t];
    if (S <= qmin && S >= 2 && S <= 16) {
      for (int P = P_force > 0 ? P_force : (nsm / S < RW_PMAX ? nsm / S : RW_PMAX); P >= 2; --P) {
        if (P > R) continue;
        if (!rows_try(d, q, R, r, S, P, smem_optin, pl)) continue;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = S; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(S * P); cfg.blockDim = dim3(RW_NT); cfg.dynamicSmemBytes = pl.smem;
        cfg.attrs = at; cfg.numAttrs = 1;
        int nclu = 0;
        if (cudaOccupancyMaxActiveClusters(&nclu, fn, &cfg) != cudaSuccess) { cudaGetLastError(); nclu = 0; }
        if (nclu < P) { if (P_force > 0) break; continue; }
        pl.ws_inner = align_up(sizeof(double) * (size_t)inner_tiles(R, R, 1));
        pl.ws = align_up(sizeof(double) * 2 * (size_t)S * P * pl.a.ylen) + align_up(sizeof(unsigned int) * 2 * S * P) +
                align_up(sizeof(double)) + pl.ws_inner +
                align_up(sizeof(double) * (size_t)S * P * d * pl.rm * rw_pad4(r)) +
                align_up(sizeof(double) * 2 * (size_t)P * pl.a.kpad * rw_pad4(r)) +
                align_up(sizeof(double) * 2 * (size_t)P * S * pl.a.gstride) + 256;
        return TP_OK;
      }
    }
    if (S_force > 0) break;
  }
  return TP_EUNSUPPORTED;
}

int als_rows_run(const RowsPlan& plan, const double* V, double* U, int sweeps, double reg, int reg_mode, double tol,
                 double stall, double* trace, int* info, void* ws, size_t ws_bytes, cudaStream_t st, long long* prof,
                 int prof_cta, int ns, const int* run_if) {
  if (!ws || ws_bytes < plan.ws) return TP_EWORKSPACE;
  RowsArgs a = plan.a;
  Carver cv(ws, ws_bytes);
  a.Y = cv.take<double>(2 * (size_t)a.S * a.P * a.ylen);
  a.flags = cv.take<unsigned int>(2 * (size_t)a.S * a.P);
  double* nsq = cv.take<double>(1);
  double* part = cv.take<double>(plan.ws_inner / sizeof(double));
  a.Xw = cv.take<double>((size_t)a.S * a.P * a.d * plan.rm * rw_pad4(a.r));
  a.Hg = cv.take<double>(2 * (size_t)a.P * a.kpad * rw_pad4(a.r));
  a.Ag = cv.take<double>(2 * (size_t)a.P * a.S * a.gstride);
  a.ns = ns;
  a.mc = g_rows_mc;
  a.split = g_rows_split;
  a.V = V; a.U = U; a.trace = trace; a.info = info; a.norm_sq = nsq;
  a.sweeps = sweeps; a.reg = reg; a.reg_mode = reg_mode; a.tol = tol; a.stall = stall;
  a.need_resid = (trace != nullptr) || (tol > 0.0) || (stall > -INFINITY);
  a.prof = prof; a.prof_cta = prof_cta;
  a.run_if = run_if;
  cudaError_t e = run_if ? cudaSuccess : cudaMemsetAsync(info, 0, 2 * sizeof(int), st);   // (the first kernel owns info)
  if (e != cudaSuccess) return cuda_status(e);
  e = cudaMemsetAsync(a.flags, 0, sizeof(unsigned int) * 2 * (size_t)a.S * a.P, st);
  if (e != cudaSuccess) return cuda_status(e);
  if (a.need_resid) {
    const int s = launch_inner(a.d, a.q, a.R, V, a.R, V, 1, nsq, part, st);   // ||V||^2 (cp.py:186-188)
    if (s != TP_OK) return s;
  }
  const void* fn = rows_kernel(plan.rm);
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
  if (e != cudaSuccess) return cuda_status(e);
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return cuda_status(e);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.S; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.gridDim = dim3(a.S * a.P); cfg.blockDim = dim3(RW_NT); cfg.dynamicSmemBytes = plan.smem; cfg.stream = st;
  cfg.attrs = at; cfg.numAttrs = 2;
  static const bool noncoop = getenv("TP_ALS_NONCOOP") && getenv("TP_ALS_NONCOOP")[0] == '1';
  if (noncoop) cfg.numAttrs = 1;
  void* args[] = {&a};
  return cuda_status(cudaLaunchKernelExC(&cfg, fn, args));
}

}  // namespace tp

extern "C" void tp_debug_set_als_rows_mc(int on) { tp::g_rows_mc = on; }
extern "C" void tp_debug_set_als_rows_split(int on) { tp::g_rows_split = on; }
