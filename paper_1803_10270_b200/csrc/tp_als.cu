// Fused, persistent CP-ALS (cp.cp_approx_als, cp.py:266-334) for sm_100a.
//
// One cooperative launch runs every sweep of a truncation.  CTA p owns a
// contiguous slab of the R target terms and keeps, in shared memory, the
// target factors of that slab for every mode (V_k[:, slab], transposed) and
// the cross matrices C_k[:, slab] = U_k^T V_k[:, slab] (cp.py:190-195).
// A mode update j (cp.py:311-320) is two phases separated by grid barriers:
//
//  A: finish the previous mode jp: stage U_jp (bulk async copies), C_jp[:, slab]
//     by DMMA, this CTA's share of the Gram entries G_jp = U_jp^T U_jp;
//     had = prod_{k!=j} C_k[:, slab] (cp.py:197-201); partial right-hand side
//     Y_p = V_j[:, slab] had^T by DMMA (cp.py:203), written to a per-CTA slot.
//  B: one bulk-async transaction pulls G_jp and this CTA's column slices of the
//     P partial right-hand sides; the CTA sums the slices in fixed order,
//     forms A = prod_{k!=j} G_k + lambda I (cp.py:312-315, 171-173) and inverts
//     it with a register-resident symmetric sweep (256 threads, one barrier per
//     pivot), then U_j[cols, :] = (A^-1 rhs)^T (cp.py:317).
//
// After each sweep (only if a trace or stopping rule needs it) the residual
// ||V||^2 - 2 Re sum prod C + sum prod G (cp.py:321-332) is formed identically
// in every CTA, so the stopping decision is uniform without host round trips.
// All cross-CTA reductions use a fixed order: results are bitwise
// reproducible for a fixed grid size.
#include "tp_common.cuh"
#include "tp_als_rows.cuh"
#include "tp_als_w.cuh"
#include <cooperative_groups.h>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

namespace cg = cooperative_groups;

namespace tp {

int inner_tiles(int ra, int rb, int same);
int launch_inner(int d, const int* q, int ra, const double* A, int rb, const double* B, int same,
                 double* out, double* partial, cudaStream_t st);
// size-unbounded streamed variant (tp_als_gen.cu): r > 32 or targets beyond shared memory
int als_generic_supported(int d, const int* q, int R, int r);
size_t als_generic_ws_bytes(int d, const int* q, int R, int r);
int als_generic_run(int d, const int* q, int R, const double* V, int r, double* U, int sweeps, double reg,
                    int reg_mode, double tol, double stall, double* trace, int* info, void* ws, size_t ws_bytes,
                    cudaStream_t st);

constexpr int ALS_NT = 256;
constexpr int ALS_NW = ALS_NT / 32;
constexpr int ALS_PART = 512;
constexpr int ALS_SMALL_NT8 = 512;   // als_small block size for r <= 8 (no 256-thread inverse mapping)   // doubles of scratch for split-K partial tiles / reductions

// padded shared-memory row stride: >= n and == 4 (mod 16) doubles, so DMMA
// fragment loads (4 rows x 8 columns per half-warp) hit distinct banks
__host__ __device__ inline int pad4(int n) { return n + (((4 - n % 16) + 16) % 16); }

struct AlsArgs {
  int d, R, r, sweeps, qmax, wmax, ncolmax, P;
  int q[TP_MAXD];
  long long offV[TP_MAXD], offU[TP_MAXD];
  int qs[TP_MAXD];     // padded stride of V_k[:, slab]^T rows in shared memory
  int qoff[TP_MAXD];   // shared-memory offset (doubles) of V_k[:, slab]^T
  int sumqs;
  const double* V;
  double* U;
  double* G;           // d * r * r
  double* Y;           // P (consumer) x P (producer) x ncolmax x r
  double* ovl;         // P
  const double* norm_sq;
  double* trace;
  int* info;           // {status bits, sweeps done}
  double reg;
  int reg_mode;
  double tol, stall;
  int need_resid;
  long long* prof;     // optional per-phase clock64 totals (CTA prof_cta), debug hook
  int prof_cta;
  unsigned int* bar_ctr;   // grid-barrier arrival counter (zeroed before launch)
  int dbg_skip;            // debug: bit mask of phases to skip (timing by subtraction)
  double* Xprev;           // [d][r][pad4(r)] last inverse per mode (warm start for Newton-Schulz)
  double* Upad;            // U_k with rows padded to pad4(r) (bulk-staged into conflict-free smem)
  long long offUp[TP_MAXD];
  // cluster variant (als_cluster): Pq CTAs per cluster share an R-slab, CTA b of a
  // cluster owns row block b of every mode
  int Pq, ldw, chunk, nbmax;
  int qoffc[TP_MAXD];      // shared-memory offset of V_k[block rows, slab] ([s][c], stride ldw)
  int ns_max;              // Newton-Schulz iterations before falling back to the exact sweep
  int clustered;           // als_persistent launched as ONE cluster of P CTAs: cluster barriers
  int local_gram;          // als_persistent: every CTA forms the whole Gram of the pending mode
  int early_inv;           // als_persistent, r <= 16: exact A_j^-1 formed in phase A by warps 0-3
  // in-kernel target: V = [A | term-major scale * L(w)], w = [ws0 W0 | ws1 W1]
  // (mode-0 scales), assembled from the un-applied states and the operator's matrices in
  // the kernel's setup instead of reading a materialised L w (explicit.py:91-93 / 99-103)
  int rcp;                 // 1: a.V unused, V from the recipe below
  int rcp_ra, rcp_rw, rcp_nw, rcp_nt;
  const double* rcpA;      // [Q_k x ra] mode-major
  const double* rcpW[2];   // [Q_k x rw] mode-major
  double rcp_ws[2];
  const double* rcp_w0;    // [nt] scale * weight (mode 0), device
  const long long* rcp_moff;   // [nt][d] matrix element offsets, -1 = identity, device
  const double* rcp_mats;
};

// The whole recipe target into dst (mode k at rows qo[k], row stride ldd) by the CTA's
// NTHR threads: (1) A blocks copied and the scaled w blocks of every mode staged in tmp
// (one global round trip for all modes); (2) identity segments copied from tmp, operator
// segments as matvecs with the matrix rows read straight from global memory (independent
// loads, unrolled).  Same products, same sequential fma order as cp.concat +
// cp_apply_kernel: bitwise equal to the materialised target.  Per-element fallback
// (rcp_value) when the w blocks do not fit tmp.
__device__ double rcp_value(const AlsArgs& a, int k, int s, int c);
template <int NTHR>
__device__ void rcp_fill(const AlsArgs& a, double* dst, int ldd, const int* qo, double* tmp, int tmp_cap) {
  const int d = a.d, ra = a.rcp_ra, rw = a.rcp_rw, wt = a.rcp_nw * a.rcp_rw, tid = threadIdx.x;
  int sumq = 0;
  for (int k = 0; k < d; ++k) sumq += a.q[k];
  if (sumq * wt > tmp_cap) {
    const int R = ra + a.rcp_nt * wt;
    for (int k = 0; k < d; ++k)
      for (int e = tid; e < a.q[k] * R; e += NTHR)
        dst[(size_t)(qo[k] + e / R) * ldd + e % R] = rcp_value(a, k, e / R, e % R);
    __syncthreads();
    return;
  }
  long long oA = 0, oW = 0;
  int ot = 0;
  for (int k = 0; k < d; ++k) {
    const int Q = a.q[k];
    for (int e = tid; e < Q * wt; e += NTHR) {
      const int u = e / wt, l = e - u * wt, blk = l / rw, j = l - blk * rw;
      tmp[ot + e] = ((k == 0) ? a.rcp_ws[blk] : 1.0) * a.rcpW[blk][oW + (long long)u * rw + j];
    }
    for (int e = tid; e < Q * ra; e += NTHR) dst[(size_t)(qo[k] + e / ra) * ldd + e % ra] = a.rcpA[oA + e];
    oA += (long long)Q * ra; oW += (long long)Q * rw; ot += Q * wt;
  }
  __syncthreads();
  ot = 0;
  for (int k = 0; k < d; ++k) {
    const int Q = a.q[k];
    const double* tW = tmp + ot;
    for (int t = 0; t < a.rcp_nt; ++t) {
      const long long mo = a.rcp_moff[t * d + k];
      const double sc = (k == 0) ? a.rcp_w0[t] : 1.0;
      double* col = dst + (size_t)qo[k] * ldd + ra + t * wt;
      if (mo < 0) {
        for (int e = tid; e < Q * wt; e += NTHR) col[(size_t)(e / wt) * ldd + e % wt] = sc * tW[e];
        continue;
      }
      for (int e = tid; e < Q * wt; e += NTHR) {
        const int sr = e / wt, l = e - sr * wt;
        const double* E = a.rcp_mats + mo + (long long)sr * Q;
        double acc = 0.0;
#pragma unroll 8
        for (int u = 0; u < Q; ++u) acc = fma(__ldg(E + u), tW[u * wt + l], acc);
        col[(size_t)sr * ldd + l] = sc * acc;
      }
    }
    ot += Q * wt;
  }
  __syncthreads();
}

// V_k[s][c] of the recipe target, bitwise equal to the materialised one (cp.concat of w,
// then cp_apply_kernel: same scale products, same sequential fma order of the matvec)
__device__ inline double rcp_value(const AlsArgs& a, int k, int s, int c) {
  long long oA = 0, oW = 0;
  for (int kk = 0; kk < k; ++kk) { oA += (long long)a.q[kk] * a.rcp_ra; oW += (long long)a.q[kk] * a.rcp_rw; }
  if (c < a.rcp_ra) return a.rcpA[oA + (long long)s * a.rcp_ra + c];
  c -= a.rcp_ra;
  const int wt = a.rcp_nw * a.rcp_rw, t = c / wt, l = c - t * wt, blk = l / a.rcp_rw, j = l - blk * a.rcp_rw;
  const double* W = a.rcpW[blk] + oW;
  const double ws = (k == 0) ? a.rcp_ws[blk] : 1.0;
  const long long mo = a.rcp_moff[t * a.d + k];
  double v;
  if (mo < 0) {
    v = ws * W[(long long)s * a.rcp_rw + j];
  } else {
    const int Q = a.q[k];
    const double* E = a.rcp_mats + mo + (long long)s * Q;
    double acc = 0.0;
    for (int u = 0; u < Q; ++u) acc = fma(__ldg(E + u), ws * W[(long long)u * a.rcp_rw + j], acc);
    v = acc;
  }
  return ((k == 0) ? a.rcp_w0[t] : 1.0) * v;
}

struct Smem {
  uint64_t* bar;        // bar[0]: U staging / Y slices, bar[1]: Gram
  double *Us, *Vs, *Cs, *Gs, *hadT, *Am, *X0, *X1, *Rm, *pub, *rb, *vb, *part, *scal;
  int* rowmap;          // [d][qmax]: (consumer CTA << 16) | row-in-consumer
  double *inbox, *mine;  // cluster variant: reduce-scatter inbox, this CTA's partial vector
};

__host__ __device__ inline size_t stage_doubles(int qmax, int r, int ncolmax, int P) {
  // staging area shared by U_k (phase A, padded rows) and the P right-hand-side
  // slices + one Gram (phase B)
  size_t a = (size_t)qmax * pad4(r), b = (size_t)P * ncolmax * r;   // U_k padded rows | the P rhs blocks
  return a > b ? a : b;
}

__host__ __device__ inline size_t als_smem_doubles(int d, int sumqs, int r, int wmax, int ncolmax, int qmax, int P) {
  const size_t w4 = (size_t)((wmax + 3) / 4) * 4;
  return 8 + stage_doubles(qmax, r, ncolmax, P) + (size_t)wmax * sumqs + (size_t)d * r * wmax +
         (size_t)d * r * r + w4 * pad4(r) + 4 * (size_t)r * pad4(r) + 72 + 4 * (size_t)ncolmax * r + ALS_PART + 8 +
         ((size_t)d * qmax + 1) / 2 + 1;
}

__device__ inline Smem carve(double* base, const AlsArgs& a) {
  Smem s;
  size_t o = 0;
  s.bar = reinterpret_cast<uint64_t*>(base + o); o += 8;
  s.Us = base + o; o += stage_doubles(a.qmax, a.r, a.ncolmax, a.P);
  s.Vs = base + o; o += (size_t)a.wmax * a.sumqs;
  s.Cs = base + o; o += (size_t)a.d * a.r * a.wmax;
  s.Gs = base + o; o += (size_t)a.d * a.r * a.r;
  s.hadT = base + o; o += (size_t)((a.wmax + 3) / 4) * 4 * pad4(a.r);
  s.Am = base + o; o += (size_t)a.r * pad4(a.r);
  s.X0 = base + o; o += (size_t)a.r * pad4(a.r);
  s.X1 = base + o; o += (size_t)a.r * pad4(a.r);
  s.Rm = base + o; o += (size_t)a.r * pad4(a.r);
  s.pub = base + o; o += 72;
  s.rb = base + o; o += (size_t)a.ncolmax * a.r;
  s.vb = base + o; o += 3 * (size_t)a.ncolmax * a.r;
  s.part = base + o; o += ALS_PART;
  s.scal = base + o; o += 8;
  s.rowmap = reinterpret_cast<int*>(base + o);
  return s;
}

// Grid barrier: one release-add per CTA on a monotonic counter, acquire-poll
// until every CTA of this epoch arrived (cheaper than cg::grid_group::sync).
// Cross-CTA data is read through L2 (__ldcg / bulk copies), so no L1 flush.
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int& epoch) {
  __syncthreads();
  if (gridDim.x == 1) return;   // one CTA: the block barrier orders everything
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned int target = epoch * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// All-CTA barrier of als_persistent: a hardware cluster barrier (release/acquire
// at cluster scope, ~400 cycles) when the whole grid is one cluster, otherwise the
// global-memory grid barrier (~3K cycles incl. skew).  Cross-CTA data is read
// through L2 (__ldcg / bulk copies) in both cases.
__device__ __forceinline__ void all_barrier(const AlsArgs& a, unsigned int& epoch) {
  if (a.clustered) {
    // the cluster-scope release alone did not order this CTA's global stores before
    // the peers' L2 reads (stale G / ovl seen on a fresh workspace): gather the CTA's
    // stores with bar.sync, then one gpu-scope fence (as the grid barrier's release)
    __syncthreads();
    if (threadIdx.x == 0) __threadfence();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    grid_barrier(a.bar_ctr, epoch);
  }
}


// Stage U_k (Q_k x r, written by other CTAs) into sm.Us with rows padded to
// pad4(r) (conflict-free DMMA fragments): one bulk async copy of the padded
// copy Upad that phase B maintains (per-row copies serialise in the SM's copy
// unit and were 6x slower).  from_user: initial guess, plain loads from U.
__device__ void stage_u(const AlsArgs& a, const Smem& sm, int k, uint32_t& phase, bool from_user = false) {
  const int r = a.r, rh = pad4(r), Q = a.q[k];
  __syncthreads();   // previous users of sm.Us are done
  if (!from_user) {
    if (threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)(Q * rh) * 8u;
      fence_proxy_async();
      mbar_arrive_expect_tx(sm.bar, bytes);
      bulk_g2s(sm.Us, a.Upad + a.offUp[k], bytes, sm.bar);
    }
    mbar_wait(sm.bar, phase);
    phase ^= 1u;
  } else {
    const double* Uk = a.U + a.offU[k];
    for (int e = threadIdx.x; e < Q * r; e += ALS_NT) sm.Us[(e / r) * rh + e % r] = __ldcg(Uk + e);
    __syncthreads();
  }
}

// Cs[k][l][c] = sum_s U_k[s][l] V_k[s][c0 + c] (cp.py:190-195) on the DMMA
// tensor pipe: M = l, N = c, K = s.  A work item is (N tile, K range); its warp
// runs all RM/8 M tiles as independent accumulator chains; the K-range partials
// are summed in fixed order through scratch (sm.X1.., free in phase A).
// wbase/nw/barid: run on warps [wbase, wbase + nw) synchronised by named barrier
// barid (0 = the whole CTA, __syncthreads)
template <int RM>
__device__ void cross_slab(const AlsArgs& a, const Smem& sm, int k, int w, int wbase = 0, int nw = ALS_NW,
                           int barid = 0) {
  constexpr int MT = RM / 8;
  const int r = a.r, Q = a.q[k], ru = pad4(r), qs = a.qs[k];
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) - wbase, nthr = nw * 32;
  auto sync = [&]() {
    if (barid == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(barid), "r"(nthr) : "memory");
  };
  const double* vs = sm.Vs + a.qoff[k];
  double* C = sm.Cs + (size_t)k * r * a.wmax;
  double* part = sm.X1;                                   // 2 r pad4(r) doubles
  const int nt = (w + 7) / 8, ksteps = (Q + 3) / 4, cap = 2 * r * ru;
  int kp = nw / nt;
  if (kp < 1) kp = 1;
  while (kp > 1 && nt * kp * MT * 64 > cap) --kp;
  const int per = (ksteps + kp - 1) / kp;
  for (int it = warp; it < nt * kp; it += nw) {
    const int n = it / kp, q = it - n * kp;
    const int c = n * 8 + (lane >> 2);
    double acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
    const int kb = q * per, ke = min(ksteps, kb + per);
#pragma unroll 2
    for (int kk = kb; kk < ke; ++kk) {
      const int s = 4 * kk + (lane & 3);
      const bool sv = s < Q;
      const double fb = (sv && c < w) ? vs[c * qs + s] : 0.0;
      double fa[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int l = m * 8 + (lane >> 2);
        fa[m] = (sv && l < r) ? sm.Us[s * ru + l] : 0.0;
      }
#pragma unroll
      for (int m = 0; m < MT; ++m) dmma_8x8x4(acc[m][0], acc[m][1], fa[m], fb);
    }
    if (kp == 1) {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int orow = m * 8 + (lane >> 2), ocol = n * 8 + 2 * (lane & 3);
        if (orow < r) {
          if (ocol < w) C[orow * a.wmax + ocol] = acc[m][0];
          if (ocol + 1 < w) C[orow * a.wmax + ocol + 1] = acc[m][1];
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        double* pt = part + ((size_t)it * MT + m) * 64;
        pt[2 * lane] = acc[m][0];
        pt[2 * lane + 1] = acc[m][1];
      }
    }
  }
  sync();
  if (kp > 1) {
    for (int e = threadIdx.x - wbase * 32; e < nt * MT * 64; e += nthr) {
      const int n = e / (MT * 64), rem = e - n * MT * 64, m = rem >> 6, ln = (rem & 63) >> 1, h = rem & 1;
      const int orow = m * 8 + (ln >> 2), ocol = n * 8 + 2 * (ln & 3) + h;
      double acc = 0.0;
      for (int q = 0; q < kp; ++q) acc += part[((size_t)(n * kp + q) * MT + m) * 64 + 2 * ln + h];
      if (orow < r && ocol < w) C[orow * a.wmax + ocol] = acc;
    }
    sync();
  }
}

// this CTA's share of G_k = U_k^T U_k (cp.py:318): the upper 8x8 tiles are
// dealt round-robin to CTAs; each tile is one DMMA chain split over the warps.
// local: every CTA forms all tiles into its own sm.Gs (small r: cheaper than the
// global round trip after the barrier).
__device__ void gram_share(const AlsArgs& a, const Smem& sm, int k, bool local = false) {
  const int r = a.r, Q = a.q[k], ru = pad4(r), lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mt = (r + 7) / 8, ntile = mt * (mt + 1) / 2;
  double* Gk = a.G + (size_t)k * r * r;
  const int ksteps = (Q + 3) / 4, per = (ksteps + ALS_NW - 1) / ALS_NW;
  const int t0 = local ? 0 : blockIdx.x, tstep = local ? 1 : gridDim.x;
  for (int t = t0; t < ntile; t += tstep) {
    int ti = 0, rem = t;
    while (rem >= mt - ti) { rem -= mt - ti; ++ti; }
    const int tj = ti + rem, m0 = ti * 8, n0 = tj * 8;
    const int l = m0 + (lane >> 2), m = n0 + (lane >> 2);
    double acc0 = 0.0, acc1 = 0.0;
    const int kb = warp * per, ke = min(ksteps, kb + per);
    for (int kk = kb; kk < ke; ++kk) {
      const int s = 4 * kk + (lane & 3);
      const double fa = (s < Q && l < r) ? sm.Us[s * ru + l] : 0.0;
      const double fb = (s < Q && m < r) ? sm.Us[s * ru + m] : 0.0;
      dmma_8x8x4(acc0, acc1, fa, fb);
    }
    __syncthreads();
    sm.part[warp * 64 + 2 * lane] = acc0;
    sm.part[warp * 64 + 2 * lane + 1] = acc1;
    __syncthreads();
    if (threadIdx.x < 64) {
      const int ln = threadIdx.x >> 1, h = threadIdx.x & 1;
      double acc = 0.0;
      for (int w = 0; w < ALS_NW; ++w) acc += sm.part[w * 64 + threadIdx.x];
      const int orow = m0 + (ln >> 2), ocol = n0 + 2 * (ln & 3) + h;
      if (orow < r && ocol < r) {
        if (!local || blockIdx.x == 0) {
          Gk[orow * r + ocol] = acc;
          Gk[ocol * r + orow] = acc;
        }
        if (gridDim.x == 1 || local) {   // no global round trip for this CTA's own Gram
          sm.Gs[(size_t)k * r * r + orow * r + ocol] = acc;
          sm.Gs[(size_t)k * r * r + ocol * r + orow] = acc;
        }
      }
    }
  }
}

// deterministic block sum (all threads call; result valid in all threads)
template <int NT = ALS_NT>
__device__ inline double block_sum(double v, double* red) {
  const int tid = threadIdx.x;
  red[tid] = v;
  __syncthreads();
  for (int w = NT / 2; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  double out = red[0];
  __syncthreads();
  return out;
}

// A = prod_{k!=j} G_k + lambda I and A^-1 -> sm.Ai (row stride r+1).
// Symmetric sweep operator (in-place Gauss-Jordan on an SPD matrix; after
// sweeping every pivot the array holds -A^-1), element-parallel: thread t owns
// row t/8 and columns (t%8) + 8u, u < RM/8, in registers.  Symmetry gives
// column k == row k, so each pivot step publishes one row and costs one
// barrier.  Returns 1 if a pivot is not positive / finite.
template <int RM>
__device__ int gram_inverse(const AlsArgs& a, const Smem& sm, int j, double* out, int os) {
  constexpr int EPT = RM / 8;
  const int r = a.r, gs = r, gk = r * r, t = threadIdx.x;
  const int i = t >> 3, c0 = t & 7;
  double v[EPT];
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int c = c0 + 8 * u;
    double x = 0.0;
    if (i < r && c < r) {
      x = 1.0;
      for (int k = 0; k < a.d; ++k)
        if (k != j) x *= sm.Gs[(size_t)k * gk + i * gs + c];
    }
    v[u] = x;
  }
  // regulariser (cp.py:171-173): fixed lambda, or reg * max(tr A, 0) / r
  double lam = a.reg;
  if (a.reg_mode) {
#pragma unroll
    for (int u = 0; u < EPT; ++u)
      if (c0 + 8 * u == i && i < r) sm.part[i] = v[u];
    __syncthreads();
    double tr = 0.0;
    for (int q = 0; q < r; ++q) tr += sm.part[q];
    lam = a.reg * fmax(tr, 0.0) / (double)r;
  }
#pragma unroll
  for (int u = 0; u < EPT; ++u)
    if (c0 + 8 * u == i && i < r) v[u] += lam;
  if (i == 0)
#pragma unroll
    for (int u = 0; u < EPT; ++u) sm.pub[c0 + 8 * u] = v[u];
  __syncthreads();
  int bad = 0;
  for (int k = 0; k < r; ++k) {
    const double* rk = sm.pub + (k & 1) * 36;
    double* rn = sm.pub + ((k + 1) & 1) * 36;
    const double d = rk[k];
    // a zero pivot of the PSD normal matrix is a zero row/column: the reference's lstsq
    // fallback (cp.py:176-177) gives the min-norm solution, i.e. a zero row/column of the
    // pseudo-inverse -- not a failure (all-zero targets / states)
    if (d < 0.0 || !isfinite(d)) bad = 1;
    const double id = (d == 0.0) ? 0.0 : rcp_nr(d);
    const double f = (i < r ? rk[i] : 0.0) * id;   // a_ik / d  (column k == row k)
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
  return bad;
}

// A = prod_{k!=j} G_k + lambda I into sm.Am (row stride pad4(r)); returns this
// thread's partial max |A_ij|.  Thread t owns row t/8, columns t%8 + 8u.
template <int RM>
__device__ double build_a(const AlsArgs& a, const Smem& sm, int j) {
  constexpr int EPT = RM / 8;
  const int r = a.r, rr = r * r, rp = pad4(r), i = threadIdx.x >> 3, c0 = threadIdx.x & 7;
  double lam = a.reg;
  if (a.reg_mode) {   // reg * max(tr A, 0) / r  (cp.py:171-173)
    double dg = 0.0;
    if (threadIdx.x < r) {
      dg = 1.0;
      for (int k = 0; k < a.d; ++k)
        if (k != j) dg *= sm.Gs[(size_t)k * rr + threadIdx.x * r + threadIdx.x];
    }
    const double tr = block_sum(dg, sm.part);
    lam = a.reg * fmax(tr, 0.0) / (double)r;
  }
  double mx = 0.0;
  if (i < r) {
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + 8 * u;
      if (c < r) {
        double f[TP_MAXD];
#pragma unroll
        for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < a.d && k != j) ? sm.Gs[(size_t)k * rr + i * r + c] : 1.0;
        double v = 1.0;
#pragma unroll
        for (int k = 0; k < TP_MAXD; ++k) v *= f[k];
        if (c == i) v += lam;
        sm.Am[i * rp + c] = v;
        mx = fmax(mx, fabs(v));
      }
    }
  }
  __syncthreads();
  return mx;
}

// Vector solve stages: out = sum_k M[k][i] v[k] with TPO = RM/8 threads per
// output (k interleaved over the group, shuffle reduction; column access keeps
// the half-warp conflict-free).  All lanes must call (uniform loop bounds).
template <int RM>
__device__ __forceinline__ double mv_dot(const double* M, int ld, const double* v, int i, int r, int part) {
  constexpr int TPO = RM / 8, KP = 8;
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int t = 0; t < KP; t += 2) {
    const int k0 = part + TPO * t, k1 = k0 + TPO;
    if (k0 < r) s0 = fma(M[k0 * ld + i], v[k0], s0);
    if (k1 < r) s1 = fma(M[k1 * ld + i], v[k1], s1);
  }
  double acc = s0 + s1;
#pragma unroll
  for (int o = TPO / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// (sum_k M[k][i] v[k], sum_k |M[k][i] v[k]|) -- for the componentwise check
template <int RM>
__device__ __forceinline__ double2 mv_dot_abs(const double* M, int ld, const double* v, int i, int r, int part) {
  constexpr int TPO = RM / 8, KP = 8;
  double s0 = 0.0, s1 = 0.0, a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int t = 0; t < KP; t += 2) {
    const int k0 = part + TPO * t, k1 = k0 + TPO;
    if (k0 < r) { const double x = M[k0 * ld + i] * v[k0]; s0 += x; a0 += fabs(x); }
    if (k1 < r) { const double x = M[k1 * ld + i] * v[k1]; s1 += x; a1 += fabs(x); }
  }
  double acc = s0 + s1, ab = a0 + a1;
#pragma unroll
  for (int o = TPO / 2; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    ab += __shfl_xor_sync(0xffffffffu, ab, o);
  }
  return make_double2(acc, ab);
}

// Solve A_j u = b for this CTA's right-hand sides b = rows of sm.rb (cp.py:317);
// A_j is already in sm.Am (build_a) on the warm path
// -> sm.vb + 2 * ncolmax * r.  Warm path (sweep > 0): one Newton-Schulz step of
// the previous sweep's inverse X0 applied to the vectors (A is symmetric, X0 is
// used through its transpose), u = X0' (2b - A X0' b), accepted when the backward
// error is at rounding level componentwise, |b - A u|_i <= 1e-13 r (|A||u|)_i (one step
// squares |I - A X|).  Returns true then; the owned rows of X1 = 2 X0 - X0 A X0
// (next sweep's warm start) are formed in the next phase A (ns_rows).
// Otherwise (first sweep, or the check fails in this CTA) the exact
// symmetric-sweep inverse, whose owned rows are stored directly.
template <int RM>
__device__ bool solve_mode(const AlsArgs& a, const Smem& sm, int j, int sweep, int E, int& status,
                           unsigned int& ns_fail, double* xprev = nullptr, int P = 0, int p = 0) {
  constexpr int TPO = RM / 8;
  if (!xprev) { xprev = a.Xprev; P = gridDim.x; p = blockIdx.x; }   // (R-sharded kernel: its group's)
  const int r = a.r, rh = pad4(r), tid = threadIdx.x;
  const int nv = a.ncolmax * r;
  double* zb = sm.vb;
  double* yb = sm.vb + nv;
  double* ub = sm.vb + 2 * nv;
  // warm starts are double-buffered by sweep parity: this sweep reads buffer
  // (sweep & 1) and writes the other, so results do not depend on CTA timing
  double* Xn = xprev + ((size_t)((sweep + 1) & 1) * a.d + j) * r * rh;
  bool ok = false;
  // after a failed Newton-Schulz check (ill-conditioned normal equations) this CTA
  // goes straight to the exact inverse for that mode in the next sweep, then
  // retries (measured on config 3 data: a failed attempt costs ~2K cycles on top
  // of the exact path)
  const bool try_ns = !((ns_fail >> j) & 1u);
  ns_fail &= ~(1u << j);
  if (try_ns && sweep > 0 && a.ns_max > 0) {
    // stage 1: z = X0' b
    for (int base = 0; base < E * TPO; base += ALS_NT) {
      const int t = base + tid, o = t / TPO, part = t - o * TPO;
      const bool act = o < E;
      const int sc = act ? o / r : 0, i = act ? o - sc * r : 0;
      const double acc = mv_dot<RM>(sm.X0, rh, sm.rb + sc * r, i, r, part);
      if (act && part == 0) zb[o] = acc;
    }
    __syncthreads();
    // stage 2: y = 2b - A z
    for (int base = 0; base < E * TPO; base += ALS_NT) {
      const int t = base + tid, o = t / TPO, part = t - o * TPO;
      const bool act = o < E;
      const int sc = act ? o / r : 0, i = act ? o - sc * r : 0;
      const double acc = mv_dot<RM>(sm.Am, rh, zb + sc * r, i, r, part);
      if (act && part == 0) yb[o] = 2.0 * sm.rb[o] - acc;
    }
    __syncthreads();
    // stage 3: u = X0' y
    for (int base = 0; base < E * TPO; base += ALS_NT) {
      const int t = base + tid, o = t / TPO, part = t - o * TPO;
      const bool act = o < E;
      const int sc = act ? o / r : 0, i = act ? o - sc * r : 0;
      const double u = mv_dot<RM>(sm.X0, rh, yb + sc * r, i, r, part);
      if (act && part == 0) ub[o] = u;
    }
    __syncthreads();
    // stage 4: componentwise backward error |b - A u|_i <= 1e-13 r (|A| |u|)_i
    int bad = 0;
    for (int base = 0; base < E * TPO; base += ALS_NT) {
      const int t = base + tid, o = t / TPO, part = t - o * TPO;
      const bool act = o < E;
      const int sc = act ? o / r : 0, i = act ? o - sc * r : 0;
      const double2 au = mv_dot_abs<RM>(sm.Am, rh, ub + sc * r, i, r, part);
      if (act && part == 0 && !(fabs(sm.rb[o] - au.x) <= 1e-13 * (double)r * au.y)) bad = 1;
    }
    ok = !__syncthreads_or(bad);
    if (!ok) ns_fail |= 1u << j;
  }
  if (ok) return true;
  status |= gram_inverse<RM>(a, sm, j, sm.X0, rh);
  __syncthreads();
  for (int base = 0; base < E * TPO; base += ALS_NT) {
    const int t = base + tid, o = t / TPO, part = t - o * TPO;
    const bool act = o < E;
    const int sc = act ? o / r : 0, i = act ? o - sc * r : 0;
    const double u = mv_dot<RM>(sm.X0, rh, sm.rb + sc * r, i, r, part);
    if (act && part == 0) ub[o] = u;
  }
  if (a.ns_max > 0)
    for (int i0 = P - 1 - p; i0 < r; i0 += P)
      for (int c = tid; c < r; c += ALS_NT) Xn[(size_t)i0 * rh + c] = sm.X0[i0 * rh + c];
  __syncthreads();
  return false;
}

// Owned rows i == P-1-p (mod P) of the next warm start X1 = 2 X0 - X0 A X0 for
// the mode solved last (A and X0 still in shared memory), phase A of the next
// mode update (off the solve's critical path; the top CTAs own no Gram tiles).
template <int RM>
__device__ void ns_rows(const AlsArgs& a, const Smem& sm, int j, int sweep, double* xprev = nullptr, int P = 0,
                        int p = 0) {
  constexpr int TPO = RM / 8;
  if (!xprev) { xprev = a.Xprev; P = gridDim.x; p = blockIdx.x; }
  const int r = a.r, rh = pad4(r), tid = threadIdx.x;
  double* Xn = xprev + ((size_t)((sweep + 1) & 1) * a.d + j) * r * rh;
  const int i_first = P - 1 - p;
  if (i_first >= r) return;
  const int nrows = (r - 1 - i_first) / P + 1;     // rows i_first, i_first + P, ...
  // all owned rows at once, chunked so the X0 A rows fit the scratch (sm.Rm: r x pad4(r))
  for (int c0 = 0; c0 < nrows; c0 += r) {
    const int nr = min(r, nrows - c0);
    double* xr = sm.Rm;                          // [nr][rh]: rows of X0 A
    for (int base = 0; base < nr * r * TPO; base += ALS_NT) {
      const int t = base + tid, o = t / TPO, part = t - o * TPO;
      const bool act = o < nr * r;
      const int q = act ? o / r : 0, c = act ? o - q * r : 0;
      const int i0 = i_first + (c0 + q) * P;
      const double acc = mv_dot<RM>(sm.Am, rh, sm.X0 + (act ? i0 : i_first) * rh, c, r, part);
      if (act && part == 0) xr[q * rh + c] = acc;
    }
    __syncthreads();
    for (int base = 0; base < nr * r * TPO; base += ALS_NT) {
      const int t = base + tid, o = t / TPO, part = t - o * TPO;
      const bool act = o < nr * r;
      const int q = act ? o / r : 0, c = act ? o - q * r : 0;
      const int i0 = i_first + (c0 + q) * P;
      const double acc = mv_dot<RM>(sm.X0, rh, xr + q * rh, c, r, part);
      if (act && part == 0) Xn[(size_t)i0 * rh + c] = 2.0 * sm.X0[i0 * rh + c] - acc;
    }
    __syncthreads();
  }
}

// Early-inverse path (als_persistent, r <= 16): warps 0-3 form the whole Gram of
// mode k from the staged U (one 8x8 upper tile per warp, full K chain) into
// sm.Gs[k]; named barrier 2 over those 128 threads.
template <int RM>
__device__ void gram_local_w4(const AlsArgs& a, const Smem& sm, int k) {
  const int r = a.r, Q = a.q[k], ru = pad4(r), lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mt = (r + 7) / 8, ntile = mt * (mt + 1) / 2;
  double* G = sm.Gs + (size_t)k * r * r;
  for (int t = warp; t < ntile; t += 4) {
    int ti = 0, rem = t;
    while (rem >= mt - ti) { rem -= mt - ti; ++ti; }
    const int tj = ti + rem, l = ti * 8 + (lane >> 2), m = tj * 8 + (lane >> 2);
    double acc0 = 0.0, acc1 = 0.0;
    const int ksteps = (Q + 3) / 4;
#pragma unroll 4
    for (int kk = 0; kk < ksteps; ++kk) {
      const int s = 4 * kk + (lane & 3);
      const double fa = (s < Q && l < r) ? sm.Us[s * ru + l] : 0.0;
      const double fb = (s < Q && m < r) ? sm.Us[s * ru + m] : 0.0;
      dmma_8x8x4(acc0, acc1, fa, fb);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int orow = ti * 8 + (lane >> 2), ocol = tj * 8 + 2 * (lane & 3) + h;
      const double v = h ? acc1 : acc0;
      if (orow < r && ocol < r) { G[orow * r + ocol] = v; G[ocol * r + orow] = v; }
    }
  }
  asm volatile("bar.sync 2, 128;" ::: "memory");
}

// gram_inverse on the 128 threads of warps 0-3 (RM <= 16: thread t owns row t/8,
// columns t%8 + 8u), named barrier 2 instead of the block barrier
template <int RM>
__device__ int gram_inverse_w4(const AlsArgs& a, const Smem& sm, int j, double* out, int os) {
  constexpr int EPT = RM / 8;
  const int r = a.r, gk = r * r, t = threadIdx.x;
  const int i = t >> 3, c0 = t & 7;
  double v[EPT];
#pragma unroll
  for (int u = 0; u < EPT; ++u) {
    const int c = c0 + 8 * u;
    double x = 0.0;
    if (i < r && c < r) {
      double f[TP_MAXD];
#pragma unroll
      for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < a.d && k != j) ? sm.Gs[(size_t)k * gk + i * r + c] : 1.0;
      x = 1.0;
#pragma unroll
      for (int k = 0; k < TP_MAXD; ++k) x *= f[k];
    }
    v[u] = x;
  }
  double lam = a.reg;
  if (a.reg_mode) {
#pragma unroll
    for (int u = 0; u < EPT; ++u)
      if (c0 + 8 * u == i && i < r) sm.part[i] = v[u];
    asm volatile("bar.sync 2, 128;" ::: "memory");
    double tr = 0.0;
    for (int q = 0; q < r; ++q) tr += sm.part[q];
    lam = a.reg * fmax(tr, 0.0) / (double)r;
  }
#pragma unroll
  for (int u = 0; u < EPT; ++u)
    if (c0 + 8 * u == i && i < r) v[u] += lam;
  if (i == 0)
#pragma unroll
    for (int u = 0; u < EPT; ++u) sm.pub[c0 + 8 * u] = v[u];
  asm volatile("bar.sync 2, 128;" ::: "memory");
  int bad = 0;
  for (int k = 0; k < r; ++k) {
    const double* rk = sm.pub + (k & 1) * 36;
    double* rn = sm.pub + ((k + 1) & 1) * 36;
    const double d = rk[k];
    // a zero pivot of the PSD normal matrix is a zero row/column: the reference's lstsq
    // fallback (cp.py:176-177) gives the min-norm solution, i.e. a zero row/column of the
    // pseudo-inverse -- not a failure (all-zero targets / states)
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
    asm volatile("bar.sync 2, 128;" ::: "memory");
  }
  if (i < r)
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int c = c0 + 8 * u;
      if (c < r) out[i * os + c] = -v[u];
    }
  return bad;
}

// debug phase timers: barrier-synchronised so the attribution is exact
#define PROF(ph)                                                        \
  do {                                                                  \
    if (TP_ALS_PROBES && a.prof) {                                                       \
      __syncthreads();                                                  \
      /* BAR.SYNC defers blocking to the next dependent instruction:  */ \
      /* force it with a shared load before sampling the clock        */ \
      prof_sink += *(volatile double*)sm.scal;                          \
      long long now = clock64();                                        \
      prof_acc[ph] += now - prof_t;                                     \
      prof_t = now;                                                     \
    }                                                                   \
  } while (0)

template <int RM>
__global__ void __launch_bounds__(ALS_NT, 1) als_persistent(const __grid_constant__ AlsArgs a) {
  extern __shared__ double smem[];
  long long prof_t = clock64();
  long long prof_acc[12] = {};
  double prof_sink = 0.0;
  unsigned int epoch = 0;
  const Smem sm = carve(smem, a);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p = blockIdx.x, P = gridDim.x, r = a.r, R = a.R, rr = r * r, rh = pad4(r);
  const int c0 = (int)((long long)R * p / P), c1 = (int)((long long)R * (p + 1) / P), w = c1 - c0;
  const int w4 = (w + 3) / 4 * 4;
  int status = 0;
  uint32_t bphase = 0, gphase = 0, xphase = 0;
  if (tid == 0) {
    mbar_init(sm.bar, 1);
    mbar_init(sm.bar + 1, 1);
    mbar_init(sm.bar + 2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int k = 0; k < a.d; ++k)
    for (int s2 = tid; s2 < a.q[k]; s2 += ALS_NT) {
      const int Qk = a.q[k];
      const int pc = ((s2 + 1) * P + Qk - 1) / Qk - 1;       // CTA owning column s2 in phase B
      const int ii = s2 - (Qk * pc) / P;
      sm.rowmap[k * a.qmax + s2] = (pc << 16) | ii;
    }
  // zero hadT padding rows (c in [w, w4)) once
  for (int e = tid; e < (w4 - w) * rh; e += ALS_NT) sm.hadT[(size_t)w * rh + e] = 0.0;
  __syncthreads();

  // ---- setup: stage V slab (transposed, padded), crosses and Grams of the initial guess
  for (int k = 0; k < a.d; ++k) {
    const int Q = a.q[k], qs = a.qs[k];
    const double* Vk = a.V + a.offV[k];
    double* vs = sm.Vs + a.qoff[k];
    for (int e = tid; e < Q * w; e += ALS_NT) {
      const int s = e / w, c = e % w;
      vs[c * qs + s] = Vk[(size_t)s * R + c0 + c];
    }
  }
  __syncthreads();
  for (int k = 0; k < a.d; ++k) {
    stage_u(a, sm, k, bphase, true);
    cross_slab<RM>(a, sm, k, w);
    gram_share(a, sm, k);
  }
  all_barrier(a, epoch);
  for (int e = tid; e < a.d * rr; e += ALS_NT) sm.Gs[e] = __ldcg(a.G + e);
  __syncthreads();

  const double norm_sq = a.need_resid ? fmax(*a.norm_sq, 0.0) : 0.0;
  const double t_norm = sqrt(norm_sq);
  double prev = INFINITY;
  int pending = -1, done = 0, rows_mode = -1, rows_sweep = 0;
  unsigned int ns_fail = 0;   // modes whose Newton-Schulz check failed in this CTA
  const bool bulk = (r & 1) == 0;
  // single-CTA grid: the right-hand side, the Gram and the new factor stay in
  // shared memory (no Y / G / U round trips through global memory)
  const bool local = P == 1;
  bool staged = false;     // local: sm.Us already holds the pending factor (padded rows)

  // early-inverse mode (r <= 16, multi-CTA): no Newton-Schulz warm starts; phase A
  // is warp-specialised -- warps 0-3 form the Gram of the previous mode and the
  // exact inverse of A_j while warps 4-7 form the Hadamard and the partial
  // right-hand side -- so phase B is one fixed-order reduction and one mat-vec
  const bool ei = RM <= 16 && a.early_inv && !local;
  for (int sweep = 0; sweep < a.sweeps; ++sweep) {
    for (int j = 0; j < a.d; ++j) {
      if (ei) {
        PROF(0);
        if (pending >= 0) {
          stage_u(a, sm, pending, bphase);
          PROF(10);
          cross_slab<RM>(a, sm, pending, w);   // all warps (measured: the cross on warps 4-7 in
          PROF(11);                            // parallel with the inverse is slower, 490 vs 458 us)
        }
        const int Qj = a.q[j], qsj = a.qs[j];
        if (warp < 4) {
          if (pending >= 0) gram_local_w4<RM>(a, sm, pending);
          status |= gram_inverse_w4<RM>(a, sm, j, sm.X0, rh);
        } else {
          for (int e = tid - 128; e < r * w; e += ALS_NT - 128) {
            const int l = e / w, c = e - l * w;
            double f[TP_MAXD];
#pragma unroll
            for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < a.d && k != j) ? sm.Cs[((size_t)k * r + l) * a.wmax + c] : 1.0;
            double v = 1.0;
#pragma unroll
            for (int k = 0; k < TP_MAXD; ++k) v *= f[k];
            sm.hadT[c * rh + l] = v;
          }
          asm volatile("bar.sync 3, 128;" ::: "memory");
          constexpr int NT = RM / 8;
          const double* vs = sm.Vs + a.qoff[j];
          const int mt = (Qj + 7) / 8, kst = w4 / 4;
          for (int m = warp - 4; m < mt; m += ALS_NW - 4) {
            const int s = m * 8 + (lane >> 2);
            const bool srow = s < Qj;
            const int rm = srow ? sm.rowmap[j * a.qmax + s] : 0;
            const int pc = rm >> 16, ii = rm & 0xffff;
            double* yrow = a.Y + (((size_t)pc * P + p) * a.ncolmax + ii) * r;
            double acc[NT][2];
#pragma unroll
            for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
            for (int kk = 0; kk < kst; ++kk) {
              const int c = 4 * kk + (lane & 3);
              const double av = (srow && c < w) ? vs[c * qsj + s] : 0.0;
              double fb[NT];
#pragma unroll
              for (int n = 0; n < NT; ++n) {
                const int l = n * 8 + (lane >> 2);
                fb[n] = (l < r) ? sm.hadT[c * rh + l] : 0.0;
              }
#pragma unroll
              for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[n][0], acc[n][1], av, fb[n]);
            }
            if (srow) {
#pragma unroll
              for (int n = 0; n < NT; ++n) {
                const int ocol = n * 8 + 2 * (lane & 3);
                if (ocol < r) yrow[ocol] = acc[n][0];
                if (ocol + 1 < r) yrow[ocol + 1] = acc[n][1];
              }
            }
          }
        }
        PROF(2);
        all_barrier(a, epoch);
        PROF(3);
        const int s0 = (int)((long long)Qj * p / P), s1 = (int)((long long)Qj * (p + 1) / P);
        const int ncol = s1 - s0, E = ncol * r, nb = a.ncolmax * r;
        double* ystage = sm.Us;
        if (bulk) {
          if (tid == 0) {
            const uint32_t ybytes = E > 0 ? (uint32_t)(P * nb) * 8u : 0u;
            fence_proxy_async();
            mbar_arrive_expect_tx(sm.bar, ybytes);
            if (ybytes) bulk_g2s(ystage, a.Y + (size_t)p * P * nb, ybytes, sm.bar);
          }
          mbar_wait(sm.bar, bphase);
          bphase ^= 1u;
          for (int o = tid; o < E; o += ALS_NT) {
            double q0 = 0.0, q1 = 0.0;
            int q = 0;
            for (; q + 2 <= P; q += 2) { q0 += ystage[(size_t)q * nb + o]; q1 += ystage[(size_t)(q + 1) * nb + o]; }
            for (; q < P; ++q) q0 += ystage[(size_t)q * nb + o];
            sm.rb[o] = q0 + q1;
          }
        } else {
          for (int o = tid; o < E; o += ALS_NT) {
            double acc = 0.0;
            for (int q = 0; q < P; ++q) acc += __ldcg(a.Y + ((size_t)p * P + q) * nb + o);
            sm.rb[o] = acc;
          }
        }
        __syncthreads();
        PROF(5);
        {   // U_j rows = (A_j^-1 b)^T  (cp.py:317)
          constexpr int TPO = RM / 8;
          double* ub = sm.vb + 2 * a.ncolmax * r;
          for (int base = 0; base < E * TPO; base += ALS_NT) {
            const int t = base + tid, o = t / TPO, part = t - o * TPO;
            const bool act = o < E;
            const int sc = act ? o / r : 0, i = act ? o - sc * r : 0;
            const double u = mv_dot<RM>(sm.X0, rh, sm.rb + sc * r, i, r, part);
            if (act && part == 0) ub[o] = u;
          }
          __syncthreads();
          PROF(9);
          if (E > 0) {
            double* Uj = a.U + a.offU[j];
            double* Up = a.Upad + a.offUp[j];
            int nf = 0;
            for (int e = tid; e < E; e += ALS_NT) {
              const int sc = e / r, i = e - sc * r;
              const double v = ub[e];
              if (!isfinite(v)) nf = 1;
              Uj[(size_t)(s0 + sc) * r + i] = v;
              Up[(size_t)(s0 + sc) * rh + i] = v;
            }
            if (nf) atomicOr(a.info, 2);
          }
        }
        pending = j;
        PROF(6);
        all_barrier(a, epoch);
        PROF(7);
        continue;
      }
      // ---------------- phase A
      PROF(0);
      if (pending >= 0) {
        if (!(TP_ALS_PROBES && a.dbg_skip & 2) && !staged) stage_u(a, sm, pending, bphase);
        staged = false;
        PROF(10);
        if (!(TP_ALS_PROBES && a.dbg_skip & 4)) cross_slab<RM>(a, sm, pending, w);
        PROF(11);
        if (!(TP_ALS_PROBES && a.dbg_skip & 8)) gram_share(a, sm, pending, a.local_gram != 0);
      }
      if (rows_mode >= 0) {   // warm-start rows of the previous NS solve
        ns_rows<RM>(a, sm, rows_mode, rows_sweep);
        rows_mode = -1;
      }
      const bool warm_ns = sweep > 0 && a.ns_max > 0;
      if (warm_ns && bulk && tid == 0) {   // prefetch this mode's warm start under phase A
        fence_proxy_async();
        mbar_arrive_expect_tx(sm.bar + 2, (uint32_t)(r * rh) * 8u);
        bulk_g2s(sm.X0, a.Xprev + ((size_t)(sweep & 1) * a.d + j) * r * rh, (uint32_t)(r * rh) * 8u, sm.bar + 2);
      }
      PROF(1);
      const int Qj = a.q[j], qsj = a.qs[j];
      for (int e = tid; e < r * w; e += ALS_NT) {   // lanes along c: conflict-free Cs rows
        const int l = e / w, c = e - l * w;
        double f[TP_MAXD];
#pragma unroll
        for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < a.d && k != j) ? sm.Cs[((size_t)k * r + l) * a.wmax + c] : 1.0;
        double v = 1.0;
#pragma unroll
        for (int k = 0; k < TP_MAXD; ++k) v *= f[k];
        sm.hadT[c * rh + l] = v;
      }
      __syncthreads();
      if (!(TP_ALS_PROBES && a.dbg_skip & 16)) {
        // Y_p[s][l] = sum_c V_j[s][c0+c] had[l][c]: M = s, N = l, K = c (DMMA),
        // all RM/8 N tiles of an M tile as independent chains.  Stored
        // consumer-major: row s goes to the CTA pc that owns column s in phase
        // B, at YT[pc][p][s - s0(pc)][:], so every consumer later pulls one
        // contiguous block with a single bulk copy.
        constexpr int NT = RM / 8;
        const double* vs = sm.Vs + a.qoff[j];
        const int mt = (Qj + 7) / 8, kst = w4 / 4;
        for (int m = warp; m < mt; m += ALS_NW) {
          const int s = m * 8 + (lane >> 2);
          const bool srow = s < Qj;
          const int rm = srow ? sm.rowmap[j * a.qmax + s] : 0;
          const int pc = rm >> 16, ii = rm & 0xffff;
          double* yrow = local ? sm.rb + (size_t)s * r : a.Y + (((size_t)pc * P + p) * a.ncolmax + ii) * r;
          double acc[NT][2];
#pragma unroll
          for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
          for (int kk = 0; kk < kst; ++kk) {
            const int c = 4 * kk + (lane & 3);
            const double av = (srow && c < w) ? vs[c * qsj + s] : 0.0;
            double fb[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const int l = n * 8 + (lane >> 2);
              fb[n] = (l < r) ? sm.hadT[c * rh + l] : 0.0;
            }
#pragma unroll
            for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[n][0], acc[n][1], av, fb[n]);
          }
          if (srow) {
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const int ocol = n * 8 + 2 * (lane & 3);
              if (ocol + 1 < r && (r & 1) == 0) {
                *reinterpret_cast<double2*>(yrow + ocol) = make_double2(acc[n][0], acc[n][1]);
              } else {
                if (ocol < r) yrow[ocol] = acc[n][0];
                if (ocol + 1 < r) yrow[ocol + 1] = acc[n][1];
              }
            }
          }
        }
      }
      PROF(2);
      all_barrier(a, epoch);
      PROF(3);
      // ---------------- phase B
      const int s0 = (int)((long long)Qj * p / P), s1 = (int)((long long)Qj * (p + 1) / P);
      const int ncol = s1 - s0, E = ncol * r;
      const int nb = a.ncolmax * r;     // one producer's block for this consumer
      double* ystage = sm.Us;           // [q][nb]
      if (local) {
        if (warm_ns && bulk) { mbar_wait(sm.bar + 2, xphase); xphase ^= 1u; }
        if (warm_ns && !bulk)   // odd r: shared rows not 16-byte aligned for the bulk copy
          for (int e = tid; e < r * rh; e += ALS_NT)
            sm.X0[e] = __ldcg(a.Xprev + ((size_t)(sweep & 1) * a.d + j) * r * rh + e);
        __syncthreads();                // sm.rb (right-hand side) and sm.Gs complete
        if (warm_ns) build_a<RM>(a, sm, j);
      } else if (bulk) {
        if (tid == 0) {
          const uint32_t gbytes = (pending >= 0 && !a.local_gram) ? (uint32_t)rr * 8u : 0u;
          const uint32_t ybytes = (E > 0 && !(TP_ALS_PROBES && a.dbg_skip & 32)) ? (uint32_t)(P * nb) * 8u : 0u;
          fence_proxy_async();
          mbar_arrive_expect_tx(sm.bar + 1, gbytes);
          if (gbytes) bulk_g2s(sm.Gs + (size_t)pending * rr, a.G + (size_t)pending * rr, gbytes, sm.bar + 1);
          mbar_arrive_expect_tx(sm.bar, ybytes);
          if (ybytes) bulk_g2s(ystage, a.Y + (size_t)p * P * nb, ybytes, sm.bar);
        }
        mbar_wait(sm.bar + 1, gphase);
        gphase ^= 1u;
        if (warm_ns) { mbar_wait(sm.bar + 2, xphase); xphase ^= 1u; }
        if (warm_ns) build_a<RM>(a, sm, j);   // overlaps the slice fetch
        PROF(8);
        mbar_wait(sm.bar, bphase);
        bphase ^= 1u;
        PROF(5);
        for (int o = tid; o < ((TP_ALS_PROBES && a.dbg_skip & 64) ? 0 : E); o += ALS_NT) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int q = 0;
          for (; q + 4 <= P; q += 4) {
            s0 += ystage[(size_t)q * nb + o];
            s1 += ystage[(size_t)(q + 1) * nb + o];
            s2 += ystage[(size_t)(q + 2) * nb + o];
            s3 += ystage[(size_t)(q + 3) * nb + o];
          }
          for (; q < P; ++q) s0 += ystage[(size_t)q * nb + o];
          sm.rb[o] = (s0 + s1) + (s2 + s3);
        }
      } else {
        if (pending >= 0 && !a.local_gram)
          for (int e = tid; e < rr; e += ALS_NT) sm.Gs[(size_t)pending * rr + e] = __ldcg(a.G + (size_t)pending * rr + e);
        if (sweep > 0 && a.ns_max > 0)
          for (int e = tid; e < r * rh; e += ALS_NT)
            sm.X0[e] = __ldcg(a.Xprev + ((size_t)(sweep & 1) * a.d + j) * r * rh + e);
        for (int o = tid; o < E; o += ALS_NT) {
          double acc = 0.0;
          for (int q = 0; q < P; ++q) acc += __ldcg(a.Y + ((size_t)p * P + q) * nb + o);
          sm.rb[o] = acc;
        }
        __syncthreads();
        if (warm_ns) build_a<RM>(a, sm, j);
      }
      __syncthreads();
      PROF(4);
      if (!(TP_ALS_PROBES && a.dbg_skip & 1) && solve_mode<RM>(a, sm, j, sweep, E, status, ns_fail)) { rows_mode = j; rows_sweep = sweep; }
      PROF(9);
      if (E > 0) {
        const double* ub = sm.vb + 2 * a.ncolmax * r;
        double* Uj = a.U + a.offU[j];
        double* Up = a.Upad + a.offUp[j];
        int nf = 0;
        for (int e = tid; e < E; e += ALS_NT) {
          const int sc = e / r, i = e - sc * r;
          const double v = ub[e];
          if (!isfinite(v)) nf = 1;
          Uj[(size_t)(s0 + sc) * r + i] = v;
          Up[(size_t)(s0 + sc) * rh + i] = v;
          if (local) sm.Us[(size_t)(s0 + sc) * rh + i] = v;   // next phase A reads it in place
        }
        if (nf) atomicOr(a.info, 2);
        if (local) staged = true;   // (cross_slab / gram_share guard the K range: no padding rows)
      }
      pending = j;
      PROF(6);
      all_barrier(a, epoch);
      PROF(7);
    }
    done = sweep + 1;
    if (a.need_resid) {
      // finish the last mode, then residual by the Gram identity (cp.py:321-326)
      stage_u(a, sm, pending, bphase);
      cross_slab<RM>(a, sm, pending, w);
      gram_share(a, sm, pending, a.local_gram != 0 || ei);
      double ov = 0.0;
      for (int e = tid; e < r * w; e += ALS_NT) {
        const int l = e / w, c = e % w;
        double v = 1.0;
        for (int k = 0; k < a.d; ++k) v *= sm.Cs[((size_t)k * r + l) * a.wmax + c];
        ov += v;
      }
      ov = block_sum(ov, sm.part);
      if (tid == 0) a.ovl[p] = ov;
      all_barrier(a, epoch);
      for (int e = tid; e < rr; e += ALS_NT) sm.Gs[(size_t)pending * rr + e] = __ldcg(a.G + (size_t)pending * rr + e);
      pending = -1;
      __syncthreads();
      double self = 0.0;
      for (int e = tid; e < rr; e += ALS_NT) {
        double v = 1.0;
        for (int k = 0; k < a.d; ++k) v *= sm.Gs[(size_t)k * rr + e];
        self += v;
      }
      self = block_sum(self, sm.part);
      double ovt = 0.0;
      if (warp == 0) {
        for (int q = lane; q < P; q += 32) ovt += __ldcg(a.ovl + q);
        ovt = warp_sum(ovt);
        if (lane == 0) sm.scal[0] = ovt;
      }
      __syncthreads();
      ovt = sm.scal[0];
      const double resid = sqrt(fmax(norm_sq - 2.0 * ovt + self, 0.0));
      if (p == 0 && tid == 0 && a.trace) a.trace[sweep] = resid;
      __syncthreads();
      if (resid <= a.tol * t_norm) break;
      if (prev - resid < a.stall * fmax(t_norm, 1.0)) break;
      prev = resid;
    }
  }
  if (status && tid == 0 && p == 0) atomicOr(a.info, 1);
  if (p == 0 && tid == 0) a.info[1] = done;
  if (TP_ALS_PROBES && a.prof && p == a.prof_cta && tid == 0) {
    for (int q = 0; q < 12; ++q) a.prof[q] += prof_acc[q];
    if (prof_sink == 12345.0) a.prof[11] += 1;
  }
}

// ===========================================================================
// Small-problem variant (one CTA, everything resident in shared memory): the
// target V, the iterate U, all crosses C_k and Grams G_k.  A mode update is five
// CTA-synchronised passes of plain FFMA loops (the work is a few 10^4 MACs, far
// too small for the DMMA pipe or for any cross-CTA exchange):
//   1. had[c][l] = prod_{k!=j} C_k[l][c];  A_j = prod_{k!=j} G_k + lambda I
//   2. rhs[s][l] = sum_c V_j[s][c] had[c][l]            (cp.py:197-203)
//   3. A_j^-1 by the symmetric sweep (exact, cp.py:312-317)
//   4. U_j[s][i] = sum_m A^-1[i][m] rhs[s][m]
//   5. C_j[l][c] = sum_s U_j[s][l] V_j[s][c], G_j = U_j^T U_j (cp.py:318-320)
// plus the residual / stopping rule per sweep (cp.py:321-332).  Used when the
// planner's grid is one CTA and the problem fits (config 0).
// ===========================================================================

// A_j = prod_{k != j} G_k + lambda I (r <= 8) inverted by ONE warp with the
// symmetric sweep operator of gram_inverse (same pivot order and update formulas),
// elements in registers: lane t owns row t/4, columns t%4 and t%4 + 4; the pivot
// row is broadcast by shuffles instead of a shared-memory hand-off + block barrier.
// Writes A^-1 to out (row stride os); returns 1 if a pivot is not positive/finite.
__device__ int warp_sweep_inverse8(const AlsArgs& a, const double* Gs, int j, double* out, int os) {
  const int r = a.r, rr = r * r, t = threadIdx.x & 31, i = t >> 2, cq = t & 3;
  double v[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int c = cq + 4 * u;
    double x = 0.0;
    if (i < r && c < r) {
      double f[TP_MAXD];
#pragma unroll
      for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < a.d && k != j) ? Gs[(size_t)k * rr + i * r + c] : 1.0;
      x = 1.0;
#pragma unroll
      for (int k = 0; k < TP_MAXD; ++k) x *= f[k];
    }
    v[u] = x;
  }
  double lam = a.reg;
  if (a.reg_mode) {   // reg * max(tr A, 0) / r  (cp.py:171-173)
    double dg = 0.0;
#pragma unroll
    for (int u = 0; u < 2; ++u) dg += (cq + 4 * u == i && i < r) ? v[u] : 0.0;
    lam = a.reg * fmax(warp_sum(dg), 0.0) / (double)r;
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
    if (cq + 4 * u == i && i < r) v[u] += lam;
  int bad = 0;
  for (int k = 0; k < r; ++k) {
    const int srow = k << 2;
    const double rk0 = __shfl_sync(0xffffffffu, v[0], srow | cq);     // a_k,cq
    const double rk1 = __shfl_sync(0xffffffffu, v[1], srow | cq);     // a_k,cq+4
    const double ri0 = __shfl_sync(0xffffffffu, v[0], srow | (i & 3));
    const double ri1 = __shfl_sync(0xffffffffu, v[1], srow | (i & 3));
    const double dk0 = __shfl_sync(0xffffffffu, v[0], srow | (k & 3));
    const double dk1 = __shfl_sync(0xffffffffu, v[1], srow | (k & 3));
    const double dd = (k >> 2) ? dk1 : dk0;                              // a_kk
    if (dd < 0.0 || !isfinite(dd)) bad = 1;          // zero pivot: min-norm (lstsq) row, see gram_inverse
    const double id = (dd == 0.0) ? 0.0 : rcp_nr(dd);
    const double aik = (i < r) ? ((i >> 2) ? ri1 : ri0) : 0.0;          // a_ik == a_ki
    const double f = aik * id;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = cq + 4 * u;
      const double akc = u ? rk1 : rk0;
      double nv = fma(-f, akc, v[u]);
      nv = (c == k) ? f : nv;
      nv = (i == k) ? ((c == k) ? -id : akc * id) : nv;
      v[u] = nv;
    }
  }
  if (i < r)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = cq + 4 * u;
      if (c < r) out[i * os + c] = -v[u];
    }
  return bad;
}

__host__ __device__ inline size_t sm_small_doubles(int d, int sumq, int qmax, int R, int r) {
  const size_t rp = (size_t)r + 1;
  return 8 + (size_t)sumq * R + (size_t)sumq * r + (size_t)d * r * R + (size_t)d * r * r + (size_t)R * r +
         (size_t)qmax * r + 2 * r * rp + 72 + ALS_PART + 8;
}

template <int RM, int NT>
__global__ void __launch_bounds__(NT, 1) als_small(const __grid_constant__ AlsArgs a) {
  extern __shared__ double smem[];
  const int tid = threadIdx.x, d = a.d, r = a.r, R = a.R, rr = r * r, rp = r + 1;
  int sumq = 0;
  int qo[TP_MAXD + 1];
  qo[0] = 0;
  for (int k = 0; k < d; ++k) { qo[k + 1] = qo[k] + a.q[k]; }
  sumq = qo[d];
  double* Vs = smem + 8;                       // [sumq][R] (global layout)
  double* Us = Vs + (size_t)sumq * R;          // [sumq][r]
  double* Cs = Us + (size_t)sumq * r;          // [d][r][R]
  double* Gsm = Cs + (size_t)d * r * R;        // [d][r][r]
  double* had = Gsm + (size_t)d * rr;          // [R][r]
  double* rhs = had + (size_t)R * r;           // [qmax][r]
  double* Am = rhs + (size_t)a.qmax * r;       // [r][r+1]
  double* Ai = Am + (size_t)r * rp;            // [r][r+1]
  Smem sm;
  memset(&sm, 0, sizeof(sm));
  sm.Gs = Gsm;
  sm.pub = Ai + (size_t)r * rp;
  sm.part = sm.pub + 72;
  sm.scal = sm.part + ALS_PART;
  for (int e = tid; e < sumq * R; e += NT) Vs[e] = a.V[e];
  for (int e = tid; e < sumq * r; e += NT) Us[e] = a.U[e];
  __syncthreads();
  // crosses and Grams of mode k from Us / Vs
  auto refresh = [&](int k) {
    const double* Uk = Us + (size_t)qo[k] * r;
    const double* Vk = Vs + (size_t)qo[k] * R;
    const int Q = a.q[k], n1 = r * R, n2 = n1 + rr;
    for (int o = tid; o < n2; o += NT) {
      // C_k[l][c] (lanes along c) or G_k[l][m]: sum_s U[s][l] X[s][c], four
      // independent accumulators so the shared loads of 4 rows are in flight together
      const bool isc = o < n1;
      const int g = isc ? o : o - n1, w = isc ? R : r, l = g / w, c = g - l * w;
      const double* X = isc ? Vk : Uk;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int s = 0;
      for (; s + 4 <= Q; s += 4) {
        s0 = fma(Uk[s * r + l], X[(size_t)s * w + c], s0);
        s1 = fma(Uk[(s + 1) * r + l], X[(size_t)(s + 1) * w + c], s1);
        s2 = fma(Uk[(s + 2) * r + l], X[(size_t)(s + 2) * w + c], s2);
        s3 = fma(Uk[(s + 3) * r + l], X[(size_t)(s + 3) * w + c], s3);
      }
      for (; s < Q; ++s) s0 = fma(Uk[s * r + l], X[(size_t)s * w + c], s0);
      const double v = (s0 + s1) + (s2 + s3);
      if (isc) Cs[(size_t)k * n1 + o] = v;
      else Gsm[(size_t)k * rr + g] = v;
    }
  };
  for (int k = 0; k < d; ++k) refresh(k);
  __syncthreads();
  const double norm_sq = a.need_resid ? fmax(*a.norm_sq, 0.0) : 0.0;
  const double t_norm = sqrt(norm_sq);
  double prev = INFINITY;
  int status = 0, done = 0;
  long long prof_acc[6] = {}, prof_t = clock64();
  double prof_sink = 0.0;
  auto mark = [&](int ph) {   // debug phase timers (a.prof): clock64 after each block barrier
    if (TP_ALS_PROBES && a.prof) {
      prof_sink += *(volatile double*)sm.scal;
      const long long now = clock64();
      prof_acc[ph] += now - prof_t;
      prof_t = now;
    }
  };
  for (int sweep = 0; sweep < a.sweeps; ++sweep) {
    for (int j = 0; j < d; ++j) {
      const int Qj = a.q[j];
      mark(5);
      // 1. Hadamards (independent loads of the d-1 factors, then the product)
      for (int e = tid; e < r * R; e += NT) {   // lanes along c (contiguous Cs rows)
        const int l = e / R, c = e - l * R;
        double f[TP_MAXD];
#pragma unroll
        for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < d && k != j) ? Cs[((size_t)k * r + l) * R + c] : 1.0;
        double v = 1.0;
#pragma unroll
        for (int k = 0; k < TP_MAXD; ++k) v *= f[k];
        had[c * r + l] = v;
      }
      __syncthreads();
      mark(0);
      // 2. right-hand side rows; 3. the inverse.  r <= 8: warp 0 inverts A_j by the
      // symmetric sweep with shuffles while the other warps form the right-hand side
      const bool winv = RM == 8;
      const int t0 = winv ? 32 : 0;
      if (winv && tid < 32) {
        status |= warp_sweep_inverse8(a, Gsm, j, Ai, rp);
      } else {
        for (int o = tid - t0; o < Qj * r; o += NT - t0) {
          const int s = o / r, l = o - s * r;
          const double* vrow = Vs + (size_t)(qo[j] + s) * R;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int c = 0;
          for (; c + 4 <= R; c += 4) {
            s0 = fma(vrow[c], had[c * r + l], s0);
            s1 = fma(vrow[c + 1], had[(c + 1) * r + l], s1);
            s2 = fma(vrow[c + 2], had[(c + 2) * r + l], s2);
            s3 = fma(vrow[c + 3], had[(c + 3) * r + l], s3);
          }
          for (; c < R; ++c) s0 = fma(vrow[c], had[c * r + l], s0);
          rhs[o] = (s0 + s1) + (s2 + s3);
        }
      }
      __syncthreads();
      if (!winv) {
        status |= gram_inverse<RM>(a, sm, j, Ai, rp);
        __syncthreads();
      }
      mark(1);
      // 4. U_j[s][i] = sum_m A^-1[i][m] rhs[s][m]
      double* Uj = Us + (size_t)qo[j] * r;
      int nf = 0;
      for (int o = tid; o < Qj * r; o += NT) {
        const int s = o / r, i = o - s * r;
        double a0 = 0.0, a1 = 0.0;
        int m = 0;
        for (; m + 2 <= r; m += 2) {
          a0 = fma(Ai[i * rp + m], rhs[s * r + m], a0);
          a1 = fma(Ai[i * rp + m + 1], rhs[s * r + m + 1], a1);
        }
        if (m < r) a0 = fma(Ai[i * rp + m], rhs[s * r + m], a0);
        const double acc = a0 + a1;
        if (!isfinite(acc)) nf = 1;
        Uj[o] = acc;
      }
      if (nf) atomicOr(a.info, 2);
      __syncthreads();
      mark(2);
      // 5. refresh C_j, G_j
      refresh(j);
      __syncthreads();
      mark(3);
    }
    done = sweep + 1;
    if (a.need_resid) {   // residual by the Gram identity (cp.py:321-326), identical in every thread
      double ov = 0.0, self = 0.0;
      for (int e = tid; e < r * R; e += NT) {
        const int l = e / R, c = e - l * R;
        double v = 1.0;
        for (int k = 0; k < d; ++k) v *= Cs[((size_t)k * r + l) * R + c];
        ov += v;
      }
      for (int e = tid; e < rr; e += NT) {
        double v = 1.0;
        for (int k = 0; k < d; ++k) v *= Gsm[(size_t)k * rr + e];
        self += v;
      }
      ov = block_sum<NT>(ov, sm.part);
      self = block_sum<NT>(self, sm.part);
      const double resid = sqrt(fmax(norm_sq - 2.0 * ov + self, 0.0));
      if (tid == 0 && a.trace) a.trace[sweep] = resid;
      if (resid <= a.tol * t_norm) break;
      if (prev - resid < a.stall * fmax(t_norm, 1.0)) break;
      prev = resid;
    }
  }
  for (int e = tid; e < sumq * r; e += NT) a.U[e] = Us[e];
  if (status && tid == 0) atomicOr(a.info, 1);
  if (tid == 0) a.info[1] = done;
  if (TP_ALS_PROBES && a.prof && tid == 0) {
    for (int q = 0; q < 6; ++q) a.prof[q] += prof_acc[q];
    if (prof_sink == 12345.0) a.prof[11] += 1;
  }
}

// ===========================================================================
// Tiny-problem variant for r <= 8 (config 0): one CTA of 512 threads with the
// whole problem in shared memory like als_small, but every contraction on the
// DMMA pipe over zero-padded operands (modes padded to 8-row tiles, R to a
// multiple of 8 with a conflict-free row stride, r to 8):
//   1. had[c][l] = prod_{k!=j} C_k[l][c]
//   2. rhs = V_j had (M = s, N = l, K = c split over warps 1..15)  |  warp 0:
//      A_j^-1 by the shuffle sweep (warp_sweep_inverse8)
//   3. U_j = rhs A_j^-1 (sums the K-split partials in its fragment loads)
//   4. C_j = U_j^T V_j and G_j = U_j^T U_j (one warp per 8-column tile)
// Four block barriers per mode update; same algorithm as cp.py:311-320.
// ===========================================================================
constexpr int TINY_NT = 512, TINY_NW = TINY_NT / 32, TINY_KSMAX = 4;
constexpr int TINY_PLD = 12;   // row stride of the right-hand-side partials (2-way, not 4-way, bank use)

struct TinyDims {
  int R8, Rs, sumqp, qmaxp;
  int qp[TP_MAXD], qo[TP_MAXD];
};

__host__ __device__ inline void tiny_dims(const int* q, int d, int R, TinyDims& t) {
  t.R8 = (R + 7) & ~7;
  t.Rs = pad4(t.R8);
  t.sumqp = 0; t.qmaxp = 0;
  for (int k = 0; k < d; ++k) {
    t.qp[k] = (q[k] + 7) & ~7;
    t.qo[k] = t.sumqp;
    t.sumqp += t.qp[k];
    t.qmaxp = t.qp[k] > t.qmaxp ? t.qp[k] : t.qmaxp;
  }
}

__host__ __device__ inline size_t tiny_smem_doubles(int d, int r, const TinyDims& t) {
  return 8 + (size_t)t.sumqp * t.Rs + (size_t)t.sumqp * 8 + (size_t)d * 8 * t.Rs + (size_t)d * r * r +
         (size_t)t.R8 * 8 + (size_t)TINY_KSMAX * t.qmaxp * TINY_PLD + 64 + ALS_PART + 8;
}

// DC: compile-time mode count (0: a.d) -- the per-mode loops unroll.
template <int DC>
__global__ void __launch_bounds__(TINY_NT, 1) als_tiny8(const __grid_constant__ AlsArgs a) {
  extern __shared__ double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int d = DC ? DC : a.d, r = a.r, R = a.R, rr = r * r;
  TinyDims td;
  tiny_dims(a.q, d, R, td);
  const int Rs = td.Rs, R8 = td.R8;
  double* scal = smem;                               // [8]
  double* Vs = smem + 8;                             // [sumqp][Rs]
  double* Us = Vs + (size_t)td.sumqp * Rs;           // [sumqp][8]
  double* Cs = Us + (size_t)td.sumqp * 8;            // [d][8][Rs]
  double* Gsm = Cs + (size_t)d * 8 * Rs;             // [d][r][r]
  double* had = Gsm + (size_t)d * rr;                // [R8][8]
  double* part = had + (size_t)R8 * 8;               // [KS][qmaxp][TINY_PLD]
  double* Ai = part + (size_t)TINY_KSMAX * td.qmaxp * TINY_PLD;   // [8][8]
  double* red = Ai + 64;                             // [ALS_PART]
  const size_t total = tiny_smem_doubles(d, r, td);
  for (size_t e = tid; e < total; e += TINY_NT) smem[e] = 0.0;   // all padding stays zero
  __syncthreads();
  if (a.rcp) rcp_fill<TINY_NT>(a, Vs, Rs, td.qo, Cs, d * 8 * Rs);   // (Cs: free scratch until the crosses)
  for (int k = 0; k < d; ++k) {
    const int Q = a.q[k];
    const double* Vk = a.V + a.offV[k];
    if (!a.rcp)
      for (int e = tid; e < Q * R; e += TINY_NT) {
        const int s = e / R, c = e - s * R;
        Vs[(size_t)(td.qo[k] + s) * Rs + c] = Vk[e];
      }
    const double* Uk = a.U + a.offU[k];
    for (int e = tid; e < Q * r; e += TINY_NT) {
      const int s = e / r, l = e - s * r;
      Us[(td.qo[k] + s) * 8 + l] = Uk[e];
    }
  }
  __syncthreads();
  // C_k = U_k^T V_k (8 x R8 tiles) and G_k = U_k^T U_k: item n < R8/8 is C tile n,
  // item R8/8 the Gram tile; K = the padded rows of mode k
  const int ntc = R8 / 8;
  auto refresh_item = [&](int k, int n) {
    const int ks = td.qp[k] / 4;
    const double* ua = Us + (size_t)td.qo[k] * 8;
    const double* vb = (n < ntc) ? Vs + (size_t)td.qo[k] * Rs + n * 8 : ua;
    const int ldb = (n < ntc) ? Rs : 8;
    double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < ks; ++kk) {
      const int srow = 4 * kk + t4;
      dmma_8x8x4(c0, c1, ua[srow * 8 + g], vb[(size_t)srow * ldb + g]);
    }
    if (n < ntc) {
      double* crow = Cs + ((size_t)k * 8 + g) * Rs + n * 8 + 2 * t4;
      crow[0] = c0; crow[1] = c1;
    } else if (g < r) {
      if (2 * t4 < r) Gsm[(size_t)k * rr + g * r + 2 * t4] = c0;
      if (2 * t4 + 1 < r) Gsm[(size_t)k * rr + g * r + 2 * t4 + 1] = c1;
    }
  };
  for (int it = warp; it < d * (ntc + 1); it += TINY_NW) refresh_item(it / (ntc + 1), it % (ntc + 1));
  __syncthreads();
  const double norm_sq = a.need_resid ? fmax(*a.norm_sq, 0.0) : 0.0;
  const double t_norm = sqrt(norm_sq);
  double prev = INFINITY;
  int status = 0, done = 0;
  long long prof_acc[6] = {}, prof_t = clock64();
  double prof_sink = 0.0;
  auto mark = [&](int ph) {   // debug phase timers (a.prof): clock64 after each block barrier
    if (TP_ALS_PROBES && a.prof) {
      prof_sink += *(volatile double*)scal;
      const long long now = clock64();
      prof_acc[ph] += now - prof_t;
      prof_t = now;
    }
  };
  // K splits of the right-hand side of mode j (warps 1.. share M tiles x K ranges)
  // worker warps 1..15 (measured: keeping warp 0's sub-partition free of workers
  // shortens the inverse chain 2.97K -> 2.16K cycles but lengthens the workers' path
  // more, 2.51 -> 2.62 us per mode update)
  constexpr int NWK = TINY_NW - 1, NTK = NWK * 32;
  const bool worker = warp != 0;
  const int wk = warp - 1;
  const int tk = tid - 32;
  auto ksn_of = [&](int j) {
    const int mt = td.qp[j] / 8;
    int ksn = NWK / mt;
    return ksn < 1 ? 1 : (ksn > TINY_KSMAX ? TINY_KSMAX : ksn);
  };
  // warps 1..: had[c][l] = prod_{k != j} C_k[l][c] (rows l >= r and columns c >= R
  // are zero), a named barrier, then part[ks][s][l] = sum_c V_j[s][c] had[c][l]
  auto hadamard_rhs = [&](int j) {
    for (int e = tk; e < R8 * 8; e += NTK) {
      const int c = e >> 3, l = e & 7;
      double f[TP_MAXD];
#pragma unroll
      for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < d && k != j) ? Cs[((size_t)k * 8 + l) * Rs + c] : 1.0;
      double v = 1.0;
#pragma unroll
      for (int k = 0; k < TP_MAXD; ++k) v *= f[k];
      had[e] = v;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NTK) : "memory");
    const int mt = td.qp[j] / 8, ksn = ksn_of(j), ksteps = R8 / 4;
    const double* va = Vs + (size_t)td.qo[j] * Rs;
    for (int it = wk; it < mt * ksn; it += NWK) {
      const int m = it / ksn, ks = it - m * ksn;
      const int kb = ksteps * ks / ksn, ke = ksteps * (ks + 1) / ksn;
      const double* arow = va + (size_t)(m * 8 + g) * Rs + t4;
      const double* bcol = had + t4 * 8 + g;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll 4
      for (int kk = kb; kk < ke; ++kk) dmma_8x8x4(c0, c1, arow[4 * kk], bcol[32 * kk]);
      double* pr = part + ((size_t)ks * td.qmaxp + m * 8 + g) * TINY_PLD + 2 * t4;
      pr[0] = c0; pr[1] = c1;
    }
  };
  // Software pipeline across mode updates: the Grams of A_{j+1} are final as soon as
  // G_j is, so warp 0 forms G_j and inverts A_{j+1} while warps 1.. form C_j, the
  // Hadamard and the right-hand side of mode j+1 (named barrier among themselves).
  // Two block barriers per mode update; the inverse is off the critical path.
  if (warp == 0) status |= warp_sweep_inverse8(a, Gsm, 0, Ai, 8);
  else if (worker) hadamard_rhs(0);
  __syncthreads();
  for (int sweep = 0; sweep < a.sweeps; ++sweep) {
    for (int j = 0; j < d; ++j) {
      const int Qj = a.q[j], mt = td.qp[j] / 8, ksn = ksn_of(j);
      mark(5);
      // U_j[s][i] = sum_m rhs[s][m] A^-1[m][i]  (K = 8: two k-steps; sums the K splits)
      if (warp < mt) {
        const int s = warp * 8 + g;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int m = 4 * kk + t4;
          double av = 0.0;
          for (int ks = 0; ks < ksn; ++ks) av += part[((size_t)ks * td.qmaxp + s) * TINY_PLD + m];
          dmma_8x8x4(c0, c1, av, Ai[m * 8 + g]);
        }
        if (!isfinite(c0) || !isfinite(c1)) atomicOr(a.info, 2);
        if (s < Qj) {
          double* ur = Us + (size_t)(td.qo[j] + s) * 8 + 2 * t4;
          ur[0] = c0; ur[1] = c1;
        }
      }
      __syncthreads();
      mark(2);
      const bool more = !(sweep == a.sweeps - 1 && j == d - 1);
      const int jn = (j + 1 == d) ? 0 : j + 1;
      if (warp == 0) {
        refresh_item(j, ntc);   // G_j
        __syncwarp();
        if (more) status |= warp_sweep_inverse8(a, Gsm, jn, Ai, 8);
        if (TP_ALS_PROBES && a.prof) prof_acc[4] += clock64() - prof_t;   // warp-0 path (debug)
      } else if (worker) {
        for (int it = wk; it < ntc; it += NWK) refresh_item(j, it);   // C_j
        asm volatile("bar.sync 1, %0;" ::"r"(NTK) : "memory");
        if (more) hadamard_rhs(jn);
      }
      __syncthreads();
      mark(3);
    }
    done = sweep + 1;
    if (a.need_resid) {   // residual by the Gram identity (cp.py:321-326), identical in every thread
      double ov = 0.0, self = 0.0;
      for (int e = tid; e < r * R; e += TINY_NT) {
        const int l = e / R, c = e - l * R;
        double v = 1.0;
        for (int k = 0; k < d; ++k) v *= Cs[((size_t)k * 8 + l) * Rs + c];
        ov += v;
      }
      for (int e = tid; e < rr; e += TINY_NT) {
        double v = 1.0;
        for (int k = 0; k < d; ++k) v *= Gsm[(size_t)k * rr + e];
        self += v;
      }
      ov = block_sum<TINY_NT>(ov, red);
      self = block_sum<TINY_NT>(self, red);
      const double resid = sqrt(fmax(norm_sq - 2.0 * ov + self, 0.0));
      if (tid == 0 && a.trace) a.trace[sweep] = resid;
      if (resid <= a.tol * t_norm) break;
      if (prev - resid < a.stall * fmax(t_norm, 1.0)) break;
      prev = resid;
    }
  }
  (void)scal;
  for (int k = 0; k < d; ++k) {
    double* Uk = a.U + a.offU[k];
    for (int e = tid; e < a.q[k] * r; e += TINY_NT) {
      const int s = e / r, l = e - s * r;
      Uk[e] = Us[(td.qo[k] + s) * 8 + l];
    }
  }
  if (status && tid == 0) atomicOr(a.info, 1);
  if (tid == 0) a.info[1] = done;
  if (TP_ALS_PROBES && a.prof && tid == 0) {
    for (int q = 0; q < 6; ++q) a.prof[q] += prof_acc[q];
    if (prof_sink == 12345.0) a.prof[11] += 1;
  }
}

// ===========================================================================
// Cluster variant.  The grid is Pr clusters x Pq CTAs; cluster a owns R-slab a,
// CTA b of the cluster owns row block b of every mode.  A mode update keeps the
// two grid barriers of als_persistent but moves ~5x less data per CTA: the
// cross C_k[:, slab] = U_k^T V_k[:, slab] is summed over the Pq row blocks
// inside the cluster (TMA bulk copies between the CTAs' shared memories, fixed
// order), so each CTA stages only its block of U_k and writes only its block's
// rows of the partial right-hand side.  The upper 8x8 Gram tiles are dealt to
// clusters and reach every CTA through global memory after the next barrier.
// ===========================================================================

__host__ __device__ inline size_t cl_stage_doubles(int nbmax, int r, int ncolmax, int Pr) {
  size_t x = (size_t)(((nbmax + 3) & ~3) + 1) * pad4(r), y = (size_t)Pr * ncolmax * r;
  return x > y ? x : y;
}

__host__ __device__ inline size_t cl_smem_doubles(int d, int r, int wmax, int ldw, int sumnb, int nbmax, int ncolmax,
                                                  int Pr, int Pq, int chunk, int qmax) {
  const size_t w4 = (size_t)((wmax + 3) / 4) * 4, rh = pad4(r);
  return 8 + cl_stage_doubles(nbmax, r, ncolmax, Pr) + (size_t)sumnb * ldw + (size_t)d * r * wmax + (size_t)d * r * r +
         w4 * rh + (size_t)(Pq - 1) * chunk + (size_t)chunk + 3 * (size_t)r * rh + 72 + 4 * (size_t)ncolmax * r +
         ALS_PART + 8 + ((size_t)d * qmax + 1) / 2 + 1;
}

__device__ inline Smem carve_cl(double* base, const AlsArgs& a, int Pr) {
  Smem s;
  size_t o = 0;
  s.bar = reinterpret_cast<uint64_t*>(base + o); o += 8;
  s.Us = base + o; o += cl_stage_doubles(a.nbmax, a.r, a.ncolmax, Pr);
  s.Vs = base + o; o += (size_t)a.sumqs * a.ldw;        // sumqs holds the padded sum of block rows here
  s.Cs = base + o; o += (size_t)a.d * a.r * a.wmax;     // Cs[k]: r x w, row stride w
  s.Gs = base + o; o += (size_t)a.d * a.r * a.r;
  s.hadT = base + o; o += (size_t)((a.wmax + 3) / 4) * 4 * pad4(a.r);
  s.inbox = base + o; o += (size_t)(a.Pq - 1) * a.chunk;   // one slot per peer, a.chunk = max partial length
  s.mine = base + o; o += (size_t)a.chunk;
  s.Am = base + o; o += (size_t)a.r * pad4(a.r);
  s.X0 = base + o; o += (size_t)a.r * pad4(a.r);
  s.X1 = nullptr;
  s.Rm = base + o; o += (size_t)a.r * pad4(a.r);
  s.pub = base + o; o += 72;
  s.rb = base + o; o += (size_t)a.ncolmax * a.r;
  s.vb = base + o; o += 3 * (size_t)a.ncolmax * a.r;
  s.part = base + o; o += ALS_PART;
  s.scal = base + o; o += 8;
  s.rowmap = reinterpret_cast<int*>(base + o);
  return s;
}

// U_k rows [qb0, qb0 + nb) -> sm.Us (row stride pad4(r)): bulk copy of the padded
// copy, or plain loads from the user's U for the initial guess.  Rows
// [nb, ceil4(nb)) are zeroed (K padding of the unpredicated DMMA loads).
__device__ void cl_stage_u(const AlsArgs& a, const Smem& sm, int k, int qb0, int nb, uint32_t& phase, bool from_user,
                           const double* Uu = nullptr, const double* Upd = nullptr) {
  const int r = a.r, rh = pad4(r);
  if (!Uu) { Uu = a.U; Upd = a.Upad; }
  __syncthreads();
  if (nb > 0) {
    if (!from_user) {
      if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)(nb * rh) * 8u;
        fence_proxy_async();
        mbar_arrive_expect_tx(sm.bar, bytes);
        bulk_g2s(sm.Us, Upd + a.offUp[k] + (size_t)qb0 * rh, bytes, sm.bar);
      }
      mbar_wait(sm.bar, phase);
      phase ^= 1u;
    } else {
      const double* Uk = Uu + a.offU[k] + (size_t)qb0 * r;
      for (int e = threadIdx.x; e < nb * r; e += ALS_NT) sm.Us[(e / r) * rh + e % r] = __ldcg(Uk + e);
    }
  }
  const int nb4 = (nb + 3) & ~3;
  for (int e = threadIdx.x; e < (nb4 - nb) * rh; e += ALS_NT) sm.Us[(size_t)nb * rh + e] = 0.0;
  __syncthreads();
}

// NS independent 8x8 DMMA chains over K = 4 ksteps rows: acc[u] += A^T B_u with
// A rows at a0 + s*arow (lane column fixed), B_u rows at b[u] + s*bst[u].  Rows
// past the block are zero and out-of-range lanes read in-bounds padding that only
// feeds discarded outputs, so the loads carry no predicates.
template <int NS>
__device__ __forceinline__ void cl_chains(uint32_t a0, uint32_t arow, const uint32_t* b, const uint32_t* bst, int ksteps,
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

// C items: m tile x group of NS n tiles of C[:, :w] = U_blk^T V_blk
template <int NS>
__device__ __forceinline__ void cl_c_item(const AlsArgs& a, const Smem& sm, const double* vs, int w, int nb, int m, int n0) {
  const int r = a.r, rh = pad4(r), lane = threadIdx.x & 31, ntc = (w + 7) / 8;
  const uint32_t us32 = smem_u32(sm.Us), vs32 = smem_u32(vs);
  uint32_t b[NS], bst[NS];
#pragma unroll
  for (int u = 0; u < NS; ++u) {
    const int n = min(n0 + u, ntc - 1);
    b[u] = vs32 + 8u * (uint32_t)(n * 8 + (lane >> 2));
    bst[u] = 8u * (uint32_t)a.ldw;
  }
  double acc[NS][2];
  cl_chains<NS>(us32 + 8u * (uint32_t)(m * 8 + (lane >> 2)), 8u * (uint32_t)rh, b, bst, (nb + 3) / 4, acc);
  const int orow = m * 8 + (lane >> 2);
  if (orow >= r) return;
#pragma unroll
  for (int u = 0; u < NS; ++u)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int ocol = (n0 + u) * 8 + 2 * (lane & 3) + h;
      if (n0 + u < ntc && ocol < w) sm.mine[orow * w + ocol] = acc[u][h];
    }
}

// this CTA's partials over its nb block rows of mode k into sm.mine:
// [0, r w): C[l][c] = sum_s U[s][l] V[s][c];  then for each upper Gram tile t
// owned by this cluster (t == cid mod Pr): 64 entries of sum_s U[s][l] U[s][m]
template <int RM>
__device__ void cl_partials(const AlsArgs& a, const Smem& sm, int k, int w, int nb, int cid, int Pr) {
  const int r = a.r, rh = pad4(r), warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mtr = (r + 7) / 8, ntc = (w + 7) / 8, nG = mtr * (mtr + 1) / 2;
  const double* vs = sm.Vs + a.qoffc[k];
  int ngroups = (ALS_NW + mtr - 1) / mtr;
  if (ngroups > ntc) ngroups = ntc;
  int ns = (ntc + ngroups - 1) / ngroups;
  if (ns > 4) { ns = 4; ngroups = (ntc + 3) / 4; }
  const int nCi = mtr * ngroups, nGi = cid < nG ? (nG - 1 - cid) / Pr + 1 : 0;
  for (int it = warp; it < nCi; it += ALS_NW) {
    const int m = it / ngroups, n0 = (it - m * ngroups) * ns;
    if (ns == 4) cl_c_item<4>(a, sm, vs, w, nb, m, n0);
    else if (ns == 3) cl_c_item<3>(a, sm, vs, w, nb, m, n0);
    else if (ns == 2) cl_c_item<2>(a, sm, vs, w, nb, m, n0);
    else cl_c_item<1>(a, sm, vs, w, nb, m, n0);
  }
  // Gram tiles of this cluster: K split over the warps, partials summed in fixed order
  const int ksteps = (nb + 3) / 4, kper = (ksteps + ALS_NW - 1) / ALS_NW;
  const int kb = min(ksteps, warp * kper), ke = min(ksteps, kb + kper);
  for (int gi = 0; gi < nGi; ++gi) {
    int g = cid + gi * Pr, ti = 0;
    while (g >= mtr - ti) { g -= mtr - ti; ++ti; }
    const int tj = ti + g;
    const uint32_t us32 = smem_u32(sm.Us) + 8u * (uint32_t)(4 * kb * rh);
    const uint32_t bb[1] = {us32 + 8u * (uint32_t)(tj * 8 + (lane >> 2))}, bst[1] = {8u * (uint32_t)rh};
    double acc[1][2];
    cl_chains<1>(us32 + 8u * (uint32_t)(ti * 8 + (lane >> 2)), 8u * (uint32_t)rh, bb, bst, ke - kb, acc);
    __syncthreads();
    sm.part[warp * 64 + 2 * lane] = acc[0][0];
    sm.part[warp * 64 + 2 * lane + 1] = acc[0][1];
    __syncthreads();
    if (threadIdx.x < 64) {
      double v = 0.0;
      for (int q = 0; q < ALS_NW; ++q) v += sm.part[q * 64 + threadIdx.x];
      sm.mine[(size_t)r * w + (size_t)gi * 64 + threadIdx.x] = v;
    }
  }
  __syncthreads();
}

// Cluster all-reduce of sm.mine (C slab partial [l][c] stride w, then this
// cluster's Gram tiles) in ONE round of TMA bulk copies between the CTAs' shared
// memories: every CTA pushes its whole partial into each peer's inbox slot, then
// every CTA sums the Pq partials in fixed rank order (bitwise identical results
// in the whole cluster) into its Cs[k]; the reduced Gram tiles go to global G
// from rank 0 (consumed after the next grid barrier).  Completion is tracked by
// mbarrier sm.bar[2]; buffers are reused only after grid barriers, so no cluster
// barrier is needed.
template <int RM>
__device__ void cl_exchange(const AlsArgs& a, const Smem& sm, cg::cluster_group& cl, int k, int w, int cid, int Pr,
                            uint32_t& ph, int& rows_mode, int rows_sweep, double* Gg = nullptr,
                            double* xprev = nullptr, int Pg = 0, int pg = 0) {
  const int r = a.r, rr = r * r, Pq = a.Pq, stride = a.chunk, b = (int)cl.block_rank(), tid = threadIdx.x;
  const int mtr = (r + 7) / 8, nG = mtr * (mtr + 1) / 2, nGi = cid < nG ? (nG - 1 - cid) / Pr + 1 : 0;
  const int rw = r * w, L = rw + nGi * 64, L2 = (L + 1) & ~1;   // even: 16-byte bulk sizes
  double* Ck = sm.Cs + (size_t)k * r * a.wmax;
  const uint32_t bar_in = smem_u32(sm.bar + 2);
  __syncthreads();   // sm.mine complete
  if (tid == 0) {
    mbar_arrive_expect_tx(sm.bar + 2, 8u * (uint32_t)((Pq - 1) * L2));
    fence_proxy_async_cluster();
    for (int q = 0; q < Pq; ++q)   // my partial -> CTA q's inbox slot for source b
      if (q != b) {
        const uint32_t slot = smem_u32(sm.inbox) + 8u * (uint32_t)((b - (b > q)) * stride);
        bulk_s2cluster(mapa_u32(slot, q), sm.mine, 8u * (uint32_t)L2, mapa_u32(bar_in, q));
      }
  }
  if (rows_mode >= 0) {   // warm-start rows of the previous solve, while the peers' partials land
    ns_rows<RM>(a, sm, rows_mode, rows_sweep, xprev, Pg, pg);
    rows_mode = -1;
  }
  mbar_wait(sm.bar + 2, ph);
  ph ^= 1u;
  double* Gk = (Gg ? Gg : a.G) + (size_t)k * rr;
  for (int idx = tid; idx < L; idx += ALS_NT) {
    double v = 0.0;
    for (int src = 0; src < Pq; ++src)
      v += (src == b) ? sm.mine[idx] : sm.inbox[(size_t)(src - (src > b)) * stride + idx];
    if (idx < rw) {
      Ck[idx] = v;
    } else if (b == 0) {
      const int gi = (idx - rw) >> 6, ln = ((idx - rw) & 63) >> 1, h = (idx - rw) & 1;
      int g = cid + gi * Pr, ti = 0;
      while (g >= mtr - ti) { g -= mtr - ti; ++ti; }
      const int tj = ti + g;
      const int orow = ti * 8 + (ln >> 2), ocol = tj * 8 + 2 * (ln & 3) + h;
      if (orow < r && ocol < r) { Gk[orow * r + ocol] = v; Gk[ocol * r + orow] = v; }
    }
  }
  __syncthreads();
}

// had = prod_{k != j} C_k[:, slab] -> hadT[c][l], then the rows of block b of the
// partial right-hand side Y[s][l] = sum_c V_j[s][c] had[l][c] (M = s, N = l,
// K = c; DMMA, RM/8 independent chains per row tile), stored consumer-major
// YT[pc][cluster][row-in-pc][:] for phase B.  Shared loads use 32-bit
// addresses and no predicates (zero padding rows/columns, discarded lanes).
template <int RM>
__device__ void cl_had_y(const AlsArgs& a, const Smem& sm, int j, int w, int b, int cid, int Pr, double* Yg = nullptr) {
  if (!Yg) Yg = a.Y;
  constexpr int NT = RM / 8;
  const int r = a.r, rh = pad4(r), ldw = a.ldw, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cs32 = smem_u32(sm.Cs), ks = 8u * (uint32_t)(r * a.wmax);   // Cs[k]: r x w, stride w
  for (int e = tid; e < r * w; e += ALS_NT) {   // lanes along c: conflict-free Cs rows
    const int l = e / w, c = e - l * w;
    const uint32_t base = cs32 + 8u * (uint32_t)(l * w + c);
    double f[TP_MAXD];
#pragma unroll
    for (int k = 0; k < TP_MAXD; ++k) f[k] = (k < a.d && k != j) ? lds64(base + (uint32_t)k * ks) : 1.0;
    double v = 1.0;
#pragma unroll
    for (int k = 0; k < TP_MAXD; ++k) v *= f[k];
    sm.hadT[c * rh + l] = v;
  }
  __syncthreads();
  const int Qj = a.q[j], Pq = a.Pq, qb0 = Qj * b / Pq, nb = Qj * (b + 1) / Pq - qb0;
  const int mt = (nb + 7) / 8, kst = (w + 3) / 4;
  const uint32_t vs32 = smem_u32(sm.Vs + a.qoffc[j]), hd32 = smem_u32(sm.hadT);
  for (int m = warp; m < mt; m += ALS_NW) {
    const int s = m * 8 + (lane >> 2);
    const uint32_t arow = vs32 + 8u * (uint32_t)(s * ldw + (lane & 3));
    const uint32_t brow = hd32 + 8u * (uint32_t)((lane & 3) * rh + (lane >> 2));
    double acc[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll 2
    for (int kk = 0; kk < kst; ++kk) {
      const double av = lds64(arow + 32u * (uint32_t)kk);
      double fb[NT];
#pragma unroll
      for (int n = 0; n < NT; ++n) fb[n] = lds64(brow + 8u * (uint32_t)(4 * kk * rh + 8 * n));
#pragma unroll
      for (int n = 0; n < NT; ++n) dmma_8x8x4(acc[n][0], acc[n][1], av, fb[n]);
    }
    if (s < nb) {
      const int rm = sm.rowmap[j * a.qmax + qb0 + s];
      const int pc = rm >> 16, ii = rm & 0xffff;
      double* yrow = Yg + (((size_t)pc * Pr + cid) * a.ncolmax + ii) * r;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int ocol = n * 8 + 2 * (lane & 3);
        if (ocol + 1 < r && (r & 1) == 0) {
          *reinterpret_cast<double2*>(yrow + ocol) = make_double2(acc[n][0], acc[n][1]);
        } else {
          if (ocol < r) yrow[ocol] = acc[n][0];
          if (ocol + 1 < r) yrow[ocol + 1] = acc[n][1];
        }
      }
    }
  }
}

template <int RM>
__global__ void __launch_bounds__(ALS_NT, 1) als_cluster(const __grid_constant__ AlsArgs a) {
  extern __shared__ double smem[];
  cg::cluster_group cl = cg::this_cluster();
  long long prof_t = clock64();
  long long prof_acc[16] = {};
  double prof_sink = 0.0;
  unsigned int epoch = 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Pq = a.Pq, b = (int)cl.block_rank(), p = blockIdx.x, P = gridDim.x, cid = p / Pq, Pr = P / Pq;
  const Smem sm = carve_cl(smem, a, Pr);
  const int r = a.r, R = a.R, rr = r * r, rh = pad4(r), ldw = a.ldw;
  const int c0 = (int)((long long)R * cid / Pr), c1 = (int)((long long)R * (cid + 1) / Pr), w = c1 - c0;
  const int w4 = (w + 3) / 4 * 4;
  int status = 0;
  uint32_t bphase = 0, gphase = 0, xphase = 0, xpf = 0;
  if (tid == 0) {
    for (int q = 0; q < 5; ++q) mbar_init(sm.bar + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int k = 0; k < a.d; ++k)
    for (int s2 = tid; s2 < a.q[k]; s2 += ALS_NT) {
      const int Qk = a.q[k];
      const int pc = ((s2 + 1) * P + Qk - 1) / Qk - 1;       // CTA owning row s2 in phase B
      const int ii = s2 - (Qk * pc) / P;
      sm.rowmap[k * a.qmax + s2] = (pc << 16) | ii;
    }
  for (int e = tid; e < (w4 - w) * rh; e += ALS_NT) sm.hadT[(size_t)w * rh + e] = 0.0;
  // ---- setup: V block rows x slab columns for every mode ([s][c], stride ldw);
  // padding rows/columns stay zero
  for (int e = tid; e < a.sumqs * ldw; e += ALS_NT) sm.Vs[e] = 0.0;
  __syncthreads();
  for (int k = 0; k < a.d; ++k) {
    const int Qk = a.q[k], qb0 = Qk * b / Pq, nb = Qk * (b + 1) / Pq - qb0;
    const double* Vk = a.V + a.offV[k] + (size_t)qb0 * R + c0;
    double* vs = sm.Vs + a.qoffc[k];
    for (int e = tid; e < nb * w; e += ALS_NT) {
      const int s2 = e / w, c = e - s2 * w;
      vs[s2 * ldw + c] = Vk[(size_t)s2 * R + c];
    }
  }
  cl.sync();   // peers' mbarriers initialised before any DSMEM copy
  for (int k = 0; k < a.d; ++k) {
    const int Qk = a.q[k], qb0 = Qk * b / Pq, nb = Qk * (b + 1) / Pq - qb0;
    cl_stage_u(a, sm, k, qb0, nb, bphase, true);
    cl_partials<RM>(a, sm, k, w, nb, cid, Pr);
    int none = -1;
    cl_exchange<RM>(a, sm, cl, k, w, cid, Pr, xphase, none, 0);
  }
  grid_barrier(a.bar_ctr, epoch);
  for (int e = tid; e < a.d * rr; e += ALS_NT) sm.Gs[e] = __ldcg(a.G + e);
  __syncthreads();

  const double norm_sq = a.need_resid ? fmax(*a.norm_sq, 0.0) : 0.0;
  const double t_norm = sqrt(norm_sq);
  double prev = INFINITY;
  int pending = -1, done = 0, rows_mode = -1, rows_sweep = 0;
  unsigned int ns_fail = 0;   // modes whose Newton-Schulz check failed in this CTA
  const bool bulk = (r & 1) == 0;

  for (int sweep = 0; sweep < a.sweeps; ++sweep) {
    for (int j = 0; j < a.d; ++j) {
      // ---------------- phase A
      PROF(0);
      if (pending >= 0) {
        const int Qk = a.q[pending], qb0 = Qk * b / Pq, nb = Qk * (b + 1) / Pq - qb0;
        cl_stage_u(a, sm, pending, qb0, nb, bphase, false);
        PROF(10);
        cl_partials<RM>(a, sm, pending, w, nb, cid, Pr);
        PROF(11);
        cl_exchange<RM>(a, sm, cl, pending, w, cid, Pr, xphase, rows_mode, rows_sweep);
        PROF(12);
      }
      if (rows_mode >= 0) {
        ns_rows<RM>(a, sm, rows_mode, rows_sweep);
        rows_mode = -1;
      }
      // prefetch this mode's warm start (X0 is free once the rows are formed)
      const bool warm_ns = sweep > 0 && a.ns_max > 0;
      if (warm_ns && tid == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(sm.bar + 4, (uint32_t)(r * rh) * 8u);
        bulk_g2s(sm.X0, a.Xprev + ((size_t)(sweep & 1) * a.d + j) * r * rh, (uint32_t)(r * rh) * 8u, sm.bar + 4);
      }
      PROF(1);
      const int Qj = a.q[j];
      cl_had_y<RM>(a, sm, j, w, b, cid, Pr);
      PROF(2);
      grid_barrier(a.bar_ctr, epoch);
      PROF(3);
      // ---------------- phase B (rows [s0, s1) of mode j)
      const int s0 = (int)((long long)Qj * p / P), s1 = (int)((long long)Qj * (p + 1) / P);
      const int ncol = s1 - s0, E = ncol * r;
      const int nbk = a.ncolmax * r;
      double* ystage = sm.Us;
      if (bulk) {
        if (tid == 0) {
          const uint32_t ybytes = E > 0 ? (uint32_t)(Pr * nbk) * 8u : 0u;
          const uint32_t gbytes = pending >= 0 ? (uint32_t)rr * 8u : 0u;
          fence_proxy_async();
          mbar_arrive_expect_tx(sm.bar + 1, gbytes);
          if (gbytes) bulk_g2s(sm.Gs + (size_t)pending * rr, a.G + (size_t)pending * rr, gbytes, sm.bar + 1);
          mbar_arrive_expect_tx(sm.bar, ybytes);
          if (ybytes) bulk_g2s(ystage, a.Y + (size_t)p * Pr * nbk, ybytes, sm.bar);
        }
        mbar_wait(sm.bar + 1, gphase);
        gphase ^= 1u;
        if (warm_ns) { mbar_wait(sm.bar + 4, xpf); xpf ^= 1u; }
        if (warm_ns) build_a<RM>(a, sm, j);   // overlaps the slice fetch
        PROF(8);
        mbar_wait(sm.bar, bphase);
        bphase ^= 1u;
        PROF(5);
        for (int o = tid; o < E; o += ALS_NT) {
          double s0a = 0.0, s1a = 0.0;
          int q = 0;
          for (; q + 2 <= Pr; q += 2) {
            s0a += ystage[(size_t)q * nbk + o];
            s1a += ystage[(size_t)(q + 1) * nbk + o];
          }
          for (; q < Pr; ++q) s0a += ystage[(size_t)q * nbk + o];
          sm.rb[o] = s0a + s1a;
        }
      } else {
        if (pending >= 0)
          for (int e = tid; e < rr; e += ALS_NT) sm.Gs[(size_t)pending * rr + e] = __ldcg(a.G + (size_t)pending * rr + e);
        if (warm_ns) { mbar_wait(sm.bar + 4, xpf); xpf ^= 1u; }
        for (int o = tid; o < E; o += ALS_NT) {
          double s0a = 0.0, s1a = 0.0;
          int q = 0;
          for (; q + 2 <= Pr; q += 2) {
            s0a += __ldcg(a.Y + ((size_t)p * Pr + q) * nbk + o);
            s1a += __ldcg(a.Y + ((size_t)p * Pr + q + 1) * nbk + o);
          }
          for (; q < Pr; ++q) s0a += __ldcg(a.Y + ((size_t)p * Pr + q) * nbk + o);
          sm.rb[o] = s0a + s1a;
        }
        __syncthreads();
        if (warm_ns) build_a<RM>(a, sm, j);
      }
      __syncthreads();
      PROF(4);
      if (solve_mode<RM>(a, sm, j, sweep, E, status, ns_fail)) { rows_mode = j; rows_sweep = sweep; }
      PROF(9);
      if (E > 0) {
        const double* ub = sm.vb + 2 * a.ncolmax * r;
        double* Uj = a.U + a.offU[j];
        double* Up = a.Upad + a.offUp[j];
        int nf = 0;
        for (int e = tid; e < E; e += ALS_NT) {
          const int sc = e / r, i = e - sc * r;
          const double v = ub[e];
          if (!isfinite(v)) nf = 1;
          Uj[(size_t)(s0 + sc) * r + i] = v;
          Up[(size_t)(s0 + sc) * rh + i] = v;
        }
        if (nf) atomicOr(a.info, 2);
      }
      pending = j;
      PROF(6);
      grid_barrier(a.bar_ctr, epoch);
      PROF(7);
    }
    done = sweep + 1;
    if (a.need_resid) {
      // finish the last mode, then residual by the Gram identity (cp.py:321-326)
      const int Qk = a.q[pending], qb0 = Qk * b / Pq, nb = Qk * (b + 1) / Pq - qb0;
      cl_stage_u(a, sm, pending, qb0, nb, bphase, false);
      cl_partials<RM>(a, sm, pending, w, nb, cid, Pr);
      cl_exchange<RM>(a, sm, cl, pending, w, cid, Pr, xphase, rows_mode, rows_sweep);
      double ov = 0.0;
      if (b == 0)
        for (int e = tid; e < r * w; e += ALS_NT) {
          const int l = e / w, c = e % w;
          double v = 1.0;
          for (int k = 0; k < a.d; ++k) v *= sm.Cs[(size_t)k * r * a.wmax + l * w + c];
          ov += v;
        }
      ov = block_sum(ov, sm.part);
      if (tid == 0 && b == 0) a.ovl[cid] = ov;
      grid_barrier(a.bar_ctr, epoch);
      for (int e = tid; e < rr; e += ALS_NT) sm.Gs[(size_t)pending * rr + e] = __ldcg(a.G + (size_t)pending * rr + e);
      pending = -1;
      __syncthreads();
      double self = 0.0;
      for (int e = tid; e < rr; e += ALS_NT) {
        double v = 1.0;
        for (int k = 0; k < a.d; ++k) v *= sm.Gs[(size_t)k * rr + e];
        self += v;
      }
      self = block_sum(self, sm.part);
      double ovt = 0.0;
      if (warp == 0) {
        for (int q = lane; q < Pr; q += 32) ovt += __ldcg(a.ovl + q);
        ovt = warp_sum(ovt);
        if (lane == 0) sm.scal[0] = ovt;
      }
      __syncthreads();
      ovt = sm.scal[0];
      const double resid = sqrt(fmax(norm_sq - 2.0 * ovt + self, 0.0));
      if (p == 0 && tid == 0 && a.trace) a.trace[sweep] = resid;
      __syncthreads();
      if (resid <= a.tol * t_norm) break;
      if (prev - resid < a.stall * fmax(t_norm, 1.0)) break;
      prev = resid;
    }
  }
  if (status && tid == 0 && p == 0) atomicOr(a.info, 1);
  if (p == 0 && tid == 0) a.info[1] = done;
  if (TP_ALS_PROBES && a.prof && p == a.prof_cta && tid == 0) {
    for (int q = 0; q < 16; ++q) a.prof[q] += prof_acc[q];
    if (prof_sink == 12345.0) a.prof[11] += 1;
  }
  cl.sync();   // no CTA may exit while peers can still address its shared memory
}

// ===========================================================================
// R-sharded truncation across GPUs in ONE launch per GPU: the
// cluster kernel above, with the target's R terms split over `ngpu` ranks.
// Rank g holds its R-slab V_g (Pr clusters x Pq CTAs over it) and a replicated
// copy of U, G and the warm starts.  Per mode update the only exchange is the
// right-hand-side reduction: every rank's producers write their partials Y into
// an exchange buffer that every peer maps (CUDA IPC over NVLink / NVSwitch);
// after a cross-GPU barrier, consumer CTA p of EVERY rank bulk-copies its rows'
// slices from all ranks' buffers (rank-major, then cluster -- the cluster
// order of the single-GPU kernel), so every rank forms the identical U_j and
// the second barrier of the mode update stays GPU-local.  Y is double-buffered
// by mode-update parity: a rank can run one mode update ahead of a peer that is
// still reading.
//
// The cross-GPU barrier: every CTA of every rank adds one arrival to EVERY
// rank's 64-bit arrival counter (red.release.sys through the peer mapping) and
// polls its own rank's counter (ld.acquire.sys) -- one hop, like the single-GPU
// grid barrier.  The counters are never reset (a fast peer may already be
// counting the next launch): each launch reads its starting value from a word
// its own previous launch left in the buffer header.  A 5 s spin limit turns a
// missing peer into status bit 4 instead of a hung GPU.
//
// One launch may also hold several groups ("virtual ranks") of CTAs: the
// single-GPU test of the exchange path, co-resident by the cooperative launch.
// ===========================================================================

constexpr int TP_MAXG = 8;

struct XgGroup {
  const double* V;
  double *U, *Upad, *G, *Xprev;
  unsigned int* bar;   // group-local grid-barrier counter (zeroed per launch)
  int* info;
};

struct XgArgs {
  int ngroups, ngpu, rank0, Pg;
  int CH;                                  // partial slices per staged chunk (two chunk slots)
  long long yhalf;                         // doubles of one parity half of Y
  XgGroup grp[TP_MAXG];
  unsigned char* peer[TP_MAXG];            // every rank's exchange buffer (arrival counter | Y[2])
};

constexpr int XG_HDR = 512;   // bytes: u64 arrival counter at [0], u64 its value after this rank's last launch at [1]

__device__ __forceinline__ unsigned long long ld_acq_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acq_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// all CTAs of all ranks; xn counts this launch's cross barriers, base is the
// counter value at launch start
__device__ __forceinline__ void xg_barrier(const XgArgs& x, int g, unsigned long long base, unsigned int& xn,
                                           int& status) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++xn;
    const unsigned long long target = base + (unsigned long long)xn * (unsigned long long)(x.Pg * x.ngpu);
    const unsigned long long* mine = reinterpret_cast<const unsigned long long*>(x.peer[x.rank0 + g]);
    __threadfence();   // this CTA's partials (gathered by bar.sync) before the system-scope release
    for (int h = 0; h < x.ngpu; ++h)
      asm volatile("red.release.sys.global.add.u64 [%0], 1;\n" ::"l"(x.peer[h]) : "memory");
    const unsigned long long t0 = globaltimer();
    while (ld_acq_sys_u64(mine) < target)
      if (globaltimer() - t0 > 5000000000ull) { status |= 4; break; }
  }
  __syncthreads();
}

// group-local grid barrier (Pg CTAs)
__device__ __forceinline__ void group_barrier(unsigned int* ctr, unsigned int& epoch, int Pg) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned int target = epoch * (unsigned)Pg;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

template <int RM>
__global__ void __launch_bounds__(ALS_NT, 1) als_xg(const __grid_constant__ AlsArgs a, const __grid_constant__ XgArgs x) {
  extern __shared__ double smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  const int Pg = x.Pg, g = blockIdx.x / Pg, p = blockIdx.x - g * Pg, P = Pg;
  const int Pq = a.Pq, b = (int)cl.block_rank(), cid = p / Pq, Pr = P / Pq;
  const int ngpu = x.ngpu, rank = x.rank0 + g;
  const XgGroup& gr = x.grp[g];
  const double* Vg = gr.V;
  double* Ug = gr.U;
  double* Upg = gr.Upad;
  double* Gg = gr.G;
  double* Xpg = gr.Xprev;
  unsigned int* barg = gr.bar;
  double* Ymine = reinterpret_cast<double*>(x.peer[rank] + XG_HDR);
  const Smem sm = carve_cl(smem, a, 2 * x.CH);   // staging: max(U block rows, two chunk slots)
  const int r = a.r, R = a.R, rr = r * r, rh = pad4(r), ldw = a.ldw;
  const int c0 = (int)((long long)R * cid / Pr), c1 = (int)((long long)R * (cid + 1) / Pr), w = c1 - c0;
  const int w4 = (w + 3) / 4 * 4;
  unsigned int epoch = 0, xn = 0;   // group-barrier epochs, cross barriers of this launch
  const unsigned long long xbase = __ldcg(reinterpret_cast<const unsigned long long*>(x.peer[rank]) + 1);
  int status = 0;
  uint32_t bphase = 0, gphase = 0, xphase = 0, xpf = 0, b3phase = 0;
  if (tid == 0) {
    for (int q = 0; q < 5; ++q) mbar_init(sm.bar + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int k = 0; k < a.d; ++k)
    for (int s2 = tid; s2 < a.q[k]; s2 += ALS_NT) {
      const int Qk = a.q[k];
      const int pc = ((s2 + 1) * P + Qk - 1) / Qk - 1;
      const int ii = s2 - (Qk * pc) / P;
      sm.rowmap[k * a.qmax + s2] = (pc << 16) | ii;
    }
  for (int e = tid; e < (w4 - w) * rh; e += ALS_NT) sm.hadT[(size_t)w * rh + e] = 0.0;
  for (int e = tid; e < a.sumqs * ldw; e += ALS_NT) sm.Vs[e] = 0.0;
  __syncthreads();
  for (int k = 0; k < a.d; ++k) {
    const int Qk = a.q[k], qb0 = Qk * b / Pq, nb = Qk * (b + 1) / Pq - qb0;
    const double* Vk = Vg + a.offV[k] + (size_t)qb0 * R + c0;
    double* vs = sm.Vs + a.qoffc[k];
    for (int e = tid; e < nb * w; e += ALS_NT) {
      const int s2 = e / w, c = e - s2 * w;
      vs[s2 * ldw + c] = Vk[(size_t)s2 * R + c];
    }
  }
  cl.sync();
  for (int k = 0; k < a.d; ++k) {
    const int Qk = a.q[k], qb0 = Qk * b / Pq, nb = Qk * (b + 1) / Pq - qb0;
    cl_stage_u(a, sm, k, qb0, nb, bphase, true, Ug, Upg);
    cl_partials<RM>(a, sm, k, w, nb, cid, Pr);
    int none = -1;
    cl_exchange<RM>(a, sm, cl, k, w, cid, Pr, xphase, none, 0, Gg, Xpg, P, p);
  }
  group_barrier(barg, epoch, Pg);
  for (int e = tid; e < a.d * rr; e += ALS_NT) sm.Gs[e] = __ldcg(Gg + e);
  __syncthreads();

  int pending = -1, rows_mode = -1, rows_sweep = 0, upd = 0;
  unsigned int ns_fail = 0;
  const int nbk = a.ncolmax * r;
  for (int sweep = 0; sweep < a.sweeps; ++sweep) {
    for (int j = 0; j < a.d; ++j, ++upd) {
      const int par = upd & 1;
      // ---------------- phase A (local: this rank's R-slab)
      if (pending >= 0) {
        const int Qk = a.q[pending], qb0 = Qk * b / Pq, nb = Qk * (b + 1) / Pq - qb0;
        cl_stage_u(a, sm, pending, qb0, nb, bphase, false, Ug, Upg);
        cl_partials<RM>(a, sm, pending, w, nb, cid, Pr);
        cl_exchange<RM>(a, sm, cl, pending, w, cid, Pr, xphase, rows_mode, rows_sweep, Gg, Xpg, P, p);
      }
      if (rows_mode >= 0) {
        ns_rows<RM>(a, sm, rows_mode, rows_sweep, Xpg, P, p);
        rows_mode = -1;
      }
      const bool warm_ns = sweep > 0 && a.ns_max > 0;
      if (warm_ns && tid == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(sm.bar + 4, (uint32_t)(r * rh) * 8u);
        bulk_g2s(sm.X0, Xpg + ((size_t)(sweep & 1) * a.d + j) * r * rh, (uint32_t)(r * rh) * 8u, sm.bar + 4);
      }
      const int Qj = a.q[j];
      cl_had_y<RM>(a, sm, j, w, b, cid, Pr, Ymine + (size_t)par * x.yhalf);
      xg_barrier(x, g, xbase, xn, status);   // every rank's partials of mode j are written
      // ---------------- phase B: rows [s0, s1) of mode j from all ranks' partials
      const int s0 = (int)((long long)Qj * p / P), s1 = (int)((long long)Qj * (p + 1) / P);
      const int ncol = s1 - s0, E = ncol * r;
      double* ystage = sm.Us;
      // rows' partial slices of all ranks (rank-major, then cluster), streamed through
      // two chunk slots of CH slices (bar[0] / bar[3]); sequential fixed-order sums
      const int CH = x.CH, nchp = (Pr + CH - 1) / CH, nchunk = E > 0 ? ngpu * nchp : 0;
      auto issue = [&](int ci) {
        const int h = ci / nchp, cc = (ci - h * nchp) * CH, n = min(CH, Pr - cc);
        const double* src = reinterpret_cast<const double*>(x.peer[h] + XG_HDR) + (size_t)par * x.yhalf +
                            ((size_t)p * Pr + cc) * nbk;
        uint64_t* bb = (ci & 1) ? sm.bar + 3 : sm.bar;
        mbar_arrive_expect_tx(bb, (uint32_t)(n * nbk) * 8u);
        bulk_g2s(ystage + (size_t)(ci & 1) * CH * nbk, src, (uint32_t)(n * nbk) * 8u, bb);
      };
      if (tid == 0) {
        const uint32_t gbytes = pending >= 0 ? (uint32_t)rr * 8u : 0u;
        fence_proxy_async();
        mbar_arrive_expect_tx(sm.bar + 1, gbytes);
        if (gbytes) bulk_g2s(sm.Gs + (size_t)pending * rr, Gg + (size_t)pending * rr, gbytes, sm.bar + 1);
        if (nchunk > 0) issue(0);
        if (nchunk > 1) issue(1);
      }
      for (int o = tid; o < E; o += ALS_NT) sm.rb[o] = 0.0;
      mbar_wait(sm.bar + 1, gphase);
      gphase ^= 1u;
      if (warm_ns) { mbar_wait(sm.bar + 4, xpf); xpf ^= 1u; }
      if (warm_ns) build_a<RM>(a, sm, j);
      for (int ci = 0; ci < nchunk; ++ci) {
        if (ci & 1) { mbar_wait(sm.bar + 3, b3phase); b3phase ^= 1u; }
        else { mbar_wait(sm.bar, bphase); bphase ^= 1u; }
        const int h = ci / nchp, cc = (ci - h * nchp) * CH, n = min(CH, Pr - cc);
        const double* slot = ystage + (size_t)(ci & 1) * CH * nbk;
        for (int o = tid; o < E; o += ALS_NT) {
          double acc = sm.rb[o];
          for (int q = 0; q < n; ++q) acc += slot[(size_t)q * nbk + o];
          sm.rb[o] = acc;
        }
        __syncthreads();   // slot consumed before it is refilled
        if (tid == 0 && ci + 2 < nchunk) {
          fence_proxy_async();
          issue(ci + 2);
        }
      }
      __syncthreads();
      if (solve_mode<RM>(a, sm, j, sweep, E, status, ns_fail, Xpg, P, p)) { rows_mode = j; rows_sweep = sweep; }
      if (E > 0) {
        const double* ub = sm.vb + 2 * a.ncolmax * r;
        double* Uj = Ug + a.offU[j];
        double* Up = Upg + a.offUp[j];
        int nf = 0;
        for (int e = tid; e < E; e += ALS_NT) {
          const int sc = e / r, i = e - sc * r;
          const double v = ub[e];
          if (!isfinite(v)) nf = 1;
          Uj[(size_t)(s0 + sc) * r + i] = v;
          Up[(size_t)(s0 + sc) * rh + i] = v;
        }
        if (nf) atomicOr(gr.info, 2);
      }
      pending = j;
      group_barrier(barg, epoch, Pg);
    }
  }
  // no rank may leave (and reuse its exchange buffer in the next launch) while a
  // peer can still read its partials
  xg_barrier(x, g, xbase, xn, status);
  if (p == 0 && tid == 0)   // every CTA of this launch has read xbase (it passed the barrier above)
    reinterpret_cast<unsigned long long*>(x.peer[rank])[1] =
        xbase + (unsigned long long)xn * (unsigned long long)(x.Pg * x.ngpu);
  if (status && tid == 0) atomicOr(gr.info, status);
  if (p == 0 && tid == 0) gr.info[1] = a.sweeps;
  cl.sync();
}

struct AlsPlan {
  AlsArgs a;
  RowsPlan rows;            // variant 8: cluster-row kernel (tp_als_rows.cu)
  WPlan w;                  // variant 9: Gram-space kernel (tp_als_w.cu) with the cluster-row kernel as its fallback
  int P, rm, variant, Pr;   // variant 0: als_persistent, 1: als_cluster (P = Pr * a.Pq), 2: als_small,
                            // 3: als_persistent as one cluster of P CTAs, 5: als_tiny8 (r <= 8, one CTA)
  size_t smem, ws_inner, ws_total, ydoubles;
};

static int g_early_inv = 1;   // debug hook: early exact inverse in the clustered R-slab kernel (r <= 16)
static int g_variant = 0;   // debug hook: 0 auto, 1 force als_persistent, 2 force als_cluster, 3 force als_small,
                            // 4 force als_persistent as one cluster (grid = cluster size), 5 force als_tiny8,
                            // 7 force the streamed generic variant (tp_als_gen.cu)
static int g_cluster = 0;   // debug hook: cluster size (0 = auto)
static int g_rows = 1;      // debug hook: cluster-row kernel for large truncations (variant 8 forces it)
static int g_rows_p = 0;    // debug hook: cluster count of the cluster-row kernel (0 = auto)

static int choose_rm(int r) { return r <= 8 ? 8 : (r <= 16 ? 16 : (r <= 32 ? 32 : 0)); }

static const void* tiny8_ptr(int d) { return d == 6 ? (const void*)als_tiny8<6> : (const void*)als_tiny8<0>; }

static const void* kernel_ptr(int rm, int variant, int d = 0) {
  if (variant == 5) return tiny8_ptr(d);
  if (variant == 3) variant = 0;   // als_persistent launched as one cluster
  if (variant == 2) {
    switch (rm) {
      case 8: return (const void*)als_small<8, ALS_SMALL_NT8>;
      case 16: return (const void*)als_small<16, ALS_NT>;
      default: return (const void*)als_small<32, ALS_NT>;
    }
  }
  if (variant == 1) {
    switch (rm) {
      case 8: return (const void*)als_cluster<8>;
      case 16: return (const void*)als_cluster<16>;
      default: return (const void*)als_cluster<32>;
    }
  }
  switch (rm) {
    case 8: return (const void*)als_persistent<8>;
    case 16: return (const void*)als_persistent<16>;
    default: return (const void*)als_persistent<32>;
  }
}

static size_t ws_total_for(int d, const int* q, int r, int P, size_t ydoubles, size_t ws_inner) {
  long long nup = 0;
  for (int k = 0; k < d; ++k) nup += (long long)q[k] * pad4(r);
  return align_up(sizeof(double) * (size_t)d * r * r) + align_up(sizeof(double) * ydoubles) +
         align_up(sizeof(double) * (size_t)P) + align_up(sizeof(double)) + ws_inner + 256 +
         align_up(sizeof(double) * 2 * (size_t)d * r * pad4(r)) + align_up(sizeof(double) * (size_t)nup);
}

// cluster variant: Pq CTAs per cluster, as many clusters (R-slabs) as can be co-resident
static int plan_cluster(int d, const int* q, int R, int r, int Pq, int smem_optin, int nsm, AlsPlan& pl) {
  int qmin = q[0], qmax = 0;
  for (int k = 0; k < d; ++k) { qmin = q[k] < qmin ? q[k] : qmin; qmax = q[k] > qmax ? q[k] : qmax; }
  if (Pq < 2 || Pq > qmin || (r & 1)) return TP_EUNSUPPORTED;
  const void* fn = kernel_ptr(pl.rm, 1);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  if (Pq > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  // Pr clusters feasible (shared memory, co-residency)?  Fills pl if so.
  auto try_pr = [&](int Pr) -> bool {
    const int P = Pr * Pq, wmax = (R + Pr - 1) / Pr, ldw = pad4(wmax), ncolmax = (qmax + P - 1) / P;
    int sumnb = 0, nbmax = 0;
    for (int k = 0; k < d; ++k) {
      const int nb = (q[k] + Pq - 1) / Pq;
      sumnb += (nb + 3) & ~3;
      nbmax = nb > nbmax ? nb : nbmax;
    }
    sumnb += 8;   // slack rows: tile lanes past the last row stay in bounds
    const int mtr = (r + 7) / 8, nG = mtr * (mtr + 1) / 2;
    int chunk = r * wmax + ((nG + Pr - 1) / Pr) * 64;   // longest partial (all-to-all exchange)
    chunk += chunk & 1;
    const size_t smem = cl_smem_doubles(d, r, wmax, ldw, sumnb, nbmax, ncolmax, Pr, Pq, chunk, qmax) * sizeof(double);
    if (smem > (size_t)smem_optin) return false;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = Pq; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(P); cfg.blockDim = dim3(ALS_NT); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
    int nclu = 0;
    if (cudaOccupancyMaxActiveClusters(&nclu, fn, &cfg) != cudaSuccess) { cudaGetLastError(); nclu = 0; }
    if (nclu < Pr) return false;
    AlsArgs& a = pl.a;
    a.Pq = Pq; a.ldw = ldw; a.chunk = chunk; a.nbmax = nbmax; a.sumqs = sumnb;
    a.wmax = wmax; a.ncolmax = ncolmax; a.P = P;
    int qo = 0;
    for (int k = 0; k < d; ++k) { a.qoffc[k] = qo; qo += (((q[k] + Pq - 1) / Pq + 3) & ~3) * ldw; }
    pl.P = P; pl.Pr = Pr; pl.smem = smem; pl.variant = 1;
    pl.ydoubles = (size_t)P * Pr * ncolmax * r;
    pl.ws_total = ws_total_for(d, q, r, P, pl.ydoubles, pl.ws_inner);
    return true;
  };
  int Pr = nsm / Pq;
  if (Pr > R) Pr = R;
  for (; Pr >= 1; --Pr) {
    if (!try_pr(Pr)) continue;
    // prefer equal slabs at the same widest slab: fewer clusters whose count divides R
    // (measured on config 1: 32 x 4 CTAs with 16-column slabs 1421 us vs 33 x 4 with
    // 15/16-column slabs 1437 us per truncation)
    const int wmax = (R + Pr - 1) / Pr;
    if (R % Pr != 0)
      for (int p2 = Pr - 1; p2 >= 1 && (R + p2 - 1) / p2 == wmax; --p2)
        if (R % p2 == 0) {
          if (try_pr(p2)) return TP_OK;
          try_pr(Pr);   // restore the first feasible plan
          break;
        }
    return TP_OK;
  }
  return TP_EUNSUPPORTED;
}

static int plan_als_uncached(int d, const int* q, int R, int r, int grid, AlsPlan& pl);

// als_persistent as one cluster of Pc <= 16 CTAs (pl already holds the persistent
// plan's per-mode offsets; only the grid-dependent fields change)
static int plan_persistent_cluster(int d, const int* q, int R, int r, int Pc, int smem_optin, AlsPlan& pl) {
  if (Pc < 2 || Pc > 16 || Pc > R) return TP_EUNSUPPORTED;
  AlsArgs& a = pl.a;
  const int wmax = (R + Pc - 1) / Pc, ncolmax = (a.qmax + Pc - 1) / Pc;
  const size_t smem = als_smem_doubles(d, a.sumqs, r, wmax, ncolmax, a.qmax, Pc) * sizeof(double);
  if (smem > (size_t)smem_optin) return TP_EUNSUPPORTED;
  const void* fn = kernel_ptr(pl.rm, 0);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  if (Pc > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = Pc; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(Pc); cfg.blockDim = dim3(ALS_NT); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
  int nclu = 0;
  if (cudaOccupancyMaxActiveClusters(&nclu, fn, &cfg) != cudaSuccess) { cudaGetLastError(); nclu = 0; }
  if (nclu < 1) return TP_EUNSUPPORTED;
  int qo = 0;
  for (int k = 0; k < d; ++k) { a.qoff[k] = qo; qo += a.qs[k] * wmax; }
  a.wmax = wmax; a.ncolmax = ncolmax; a.P = Pc; a.Pq = Pc; a.clustered = 1;
  a.early_inv = (r <= 16 && g_early_inv) ? 1 : 0;
  pl.P = Pc; pl.Pr = Pc; pl.smem = smem; pl.variant = 3;
  pl.ydoubles = (size_t)Pc * Pc * ncolmax * r;
  pl.ws_total = ws_total_for(d, q, r, Pc, pl.ydoubles, pl.ws_inner);
  return TP_OK;
}

// plans are pure functions of (device, sizes, grid, debug variant): cache them, the
// cluster occupancy queries cost tens of microseconds per call
struct PlanKey {
  int dev, d, R, r, grid, variant, cluster;
  int q[TP_MAXD];
  bool operator==(const PlanKey& o) const { return memcmp(this, &o, sizeof(PlanKey)) == 0; }
};

static int plan_als(int d, const int* q, int R, int r, int grid, AlsPlan& pl) {
  if (d < 1 || R < 1 || r < 1 || !q) return TP_EINVAL;
  if (d > TP_MAXD) return TP_EUNSUPPORTED;   // (the streamed variant takes up to TP_MAXD_GEN modes)
  static std::mutex mu;
  static std::vector<std::pair<PlanKey, AlsPlan>> cache;
  PlanKey key;
  memset(&key, 0, sizeof(key));
  if (cudaGetDevice(&key.dev) != cudaSuccess) { cudaGetLastError(); key.dev = -1; }
  key.d = d; key.R = R; key.r = r; key.grid = grid; key.variant = g_variant * 2 + g_early_inv + 1000 * g_rows + 100000 * g_rows_p + 4000000 * als_w_enabled(); key.cluster = g_cluster;
  for (int k = 0; k < d; ++k) key.q[k] = q[k];
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : cache)
      if (e.first == key) { pl = e.second; return TP_OK; }
  }
  const int st = plan_als_uncached(d, q, R, r, grid, pl);
  if (st == TP_OK) {
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() > 64) cache.clear();
    cache.emplace_back(key, pl);
  }
  return st;
}

static int plan_als_uncached(int d, const int* q, int R, int r, int grid, AlsPlan& pl) {
  if (d < 1 || R < 1 || r < 1 || !q) return TP_EINVAL;
  if (d > TP_MAXD) return TP_EUNSUPPORTED;
  for (int k = 0; k < d; ++k) if (q[k] < 1) return TP_EINVAL;
  pl.rm = choose_rm(r);
  if (!pl.rm) return TP_EUNSUPPORTED;
  int dev = 0, nsm = 148, smem_optin = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  } else {
    cudaGetLastError();
  }
  if (smem_optin <= 0) smem_optin = 227 * 1024;
  int sumqs = 0, qmax = 0;
  for (int k = 0; k < d; ++k) { sumqs += pad4(q[k]); qmax = q[k] > qmax ? q[k] : qmax; }
  int P = grid;
  if (P <= 0) {
    double work = 4.0 * qmax * (double)R * r;   // flops of one mode update
    P = (int)(work / 5.0e4);   // measured: cfg3 (R=588, r=12) best at >= 32 CTAs, cfg0 at 1
    if (P < 1) P = 1;
  }
  if (P > nsm) P = nsm;
  if (P > R) P = R;
  size_t smem = 0;
  for (;;) {
    int wmax = (R + P - 1) / P, ncolmax = (qmax + P - 1) / P;
    smem = als_smem_doubles(d, sumqs, r, wmax, ncolmax, qmax, P) * sizeof(double);
    if (smem <= (size_t)smem_optin) break;
    if (P >= nsm || P >= R) return TP_EUNSUPPORTED;
    ++P;
  }
  memset(&pl.a, 0, sizeof(pl.a));
  AlsArgs& a = pl.a;
  a.d = d; a.R = R; a.r = r; a.qmax = qmax; a.sumqs = sumqs; a.P = P;
  a.wmax = (R + P - 1) / P; a.ncolmax = (qmax + P - 1) / P;
  long long ov = 0, ou = 0, oup = 0;
  int qo = 0;
  for (int k = 0; k < d; ++k) {
    a.q[k] = q[k]; a.qs[k] = pad4(q[k]); a.offV[k] = ov; a.offU[k] = ou; a.qoff[k] = qo;
    a.offUp[k] = oup;
    ov += (long long)q[k] * R; ou += (long long)q[k] * r; qo += a.qs[k] * a.wmax; oup += (long long)q[k] * pad4(r);
  }
  a.local_gram = 0;   // (r <= 16 measured slower: 3 tiles recomputed cost more than the round trip)
  a.early_inv = (r <= 16 && P > 1 && g_early_inv) ? 1 : 0;   // exact inverse formed in phase A (warps 0-3)
  pl.P = P;
  pl.smem = smem;
  pl.ws_inner = align_up(sizeof(double) * (size_t)inner_tiles(R, R, 1));
  pl.Pr = P;
  pl.variant = 0;
  pl.ydoubles = (size_t)P * P * a.ncolmax * r;
  pl.ws_total = ws_total_for(d, q, r, P, pl.ydoubles, pl.ws_inner);
  (void)oup;
  // mid-size problems: the same kernel as ONE cluster of up to 16 CTAs (hardware
  // cluster barriers instead of the global-memory grid barrier)
  if (g_variant == 4) {
    const int Pc = grid > 0 ? grid : (P < 16 ? P : 16);
    if (plan_persistent_cluster(d, q, R, r, Pc, smem_optin, pl) == TP_OK) return TP_OK;
    return TP_EUNSUPPORTED;
  }
  // measured (tools/als_cl_scan.py, tools/ei_scan.sh; with the early inverse for r <= 16):
  // one 16-CTA cluster beats the grid-barrier R-slab kernel at 12-49 CTAs -- config 3
  // (Q=64, R=588, r=12) 8.37 -> 7.60 us per mode update, (96, 200, 8) 7.89 -> 6.77,
  // (128, 300, 16) 9.26 -> 9.11
  if (g_variant == 0 && grid <= 0 && P >= 8 && P <= 64) {
    AlsPlan cp = pl;
    if (plan_persistent_cluster(d, q, R, r, 16, smem_optin, cp) == TP_OK) { pl = cp; return TP_OK; }
  }
  // large truncations: the cluster-row kernel (one flag exchange + two cluster barriers per
  // mode update instead of two grid barriers)
  if (g_variant == 8 || g_variant == 9 || (g_variant == 0 && grid <= 0 && P >= 64 && g_rows)) {
    AlsPlan cp = pl;
    if (als_rows_plan(d, q, R, r, g_cluster > 0 ? g_cluster : 0, g_rows_p, cp.rows) == TP_OK) {
      cp.variant = 8; cp.P = cp.rows.a.S * cp.rows.a.P; cp.Pr = cp.rows.a.P; cp.smem = cp.rows.smem;
      cp.ws_total = cp.rows.ws;
      // well-conditioned large truncations: the sweeps in Gram space (no reduction over the factor
      // rows), the cluster-row kernel launched behind it as the conditioning fallback
      if ((g_variant == 0 || g_variant == 9) && als_w_plan(d, q, R, r, cp.w) == TP_OK) {
        cp.variant = 9; cp.P = cp.w.a.P << cp.w.a.pair; cp.Pr = cp.w.a.P; cp.smem = cp.w.smem;
        cp.ws_total = align_up(cp.w.ws) + cp.rows.ws;
      } else if (g_variant == 9) {
        return TP_EUNSUPPORTED;
      }
      pl = cp;
      return TP_OK;
    }
    if (g_variant == 8 || g_variant == 9) return TP_EUNSUPPORTED;
  }
  // large truncations: the cluster variant (fewer bytes per CTA per mode update)
  const bool want = g_variant == 2 || (g_variant == 0 && grid <= 0 && P >= 64 && g_cluster >= 0);
  if (want) {
    AlsPlan cp = pl;
    const int sizes[3] = {8, 4, 2};
    for (int t = 0; t < 3; ++t) {
      const int Pq = g_cluster > 0 ? g_cluster : sizes[t];
      if (plan_cluster(d, q, R, r, Pq, smem_optin, nsm, cp) == TP_OK) { pl = cp; return TP_OK; }
      if (g_cluster > 0) break;
    }
    if (g_variant == 2) return TP_EUNSUPPORTED;
  }
  // tiny problems: one CTA with everything in shared memory; r <= 8 on the DMMA pipe
  if (pl.rm == 8 && (g_variant == 5 || (g_variant == 0 && grid <= 0 && P == 1))) {
    TinyDims td;
    tiny_dims(q, d, R, td);
    const size_t sm_tiny = tiny_smem_doubles(d, r, td) * sizeof(double);
    if (sm_tiny <= (size_t)smem_optin) {
      pl.variant = 5; pl.P = 1; pl.Pr = 1; pl.smem = sm_tiny;
      return TP_OK;
    }
    if (g_variant == 5) return TP_EUNSUPPORTED;
  }
  if (g_variant == 3 || (g_variant == 0 && grid <= 0 && P == 1)) {
    int sumq = 0;
    for (int k = 0; k < d; ++k) sumq += q[k];
    const size_t sm_small = sm_small_doubles(d, sumq, qmax, R, r) * sizeof(double);
    if (sm_small <= (size_t)smem_optin) {
      pl.variant = 2; pl.P = 1; pl.Pr = 1; pl.smem = sm_small;
    } else if (g_variant == 3) {
      return TP_EUNSUPPORTED;
    }
  }
  return TP_OK;
}

}  // namespace tp

using namespace tp;

static long long* g_prof = nullptr;
static int g_prof_cta = 0;
static int g_skip = 0;
static int g_ns_max = 6;

extern "C" {

// debug hook (not part of the public header): per-phase clock64 totals of CTA 0
void tp_debug_set_als_profile(long long* dev_ptr) { g_prof = dev_ptr; }
void tp_debug_set_als_profile_cta(int cta) { g_prof_cta = cta; }
// debug hook: skip phases (results are wrong) to time them by subtraction
void tp_debug_set_als_skip(int mask) { g_skip = mask; }
// debug hook: Newton-Schulz iteration cap (0 = always the exact sweep inversion)
void tp_debug_set_als_ns(int n) { g_ns_max = n; }
// debug hook: kernel variant (0 auto, 1 als_persistent, 2 als_cluster) and cluster size (0 auto, -1 never)
void tp_debug_set_als_variant(int variant, int cluster) { g_variant = variant; g_cluster = cluster; }
void tp_debug_set_als_early_inv(int on) { g_early_inv = on; }
void tp_debug_set_als_rows(int on, int nclusters) { g_rows = on; g_rows_p = nclusters; }

int tp_cp_als_plan(int d, const int* q, int R, int r, int grid, int* out) {
  if (!out) return TP_EINVAL;
  AlsPlan pl;
  const int st = g_variant == 7 ? TP_EUNSUPPORTED : plan_als(d, q, R, r, grid, pl);
  if (st == TP_EUNSUPPORTED && als_generic_supported(d, q, R, r)) {   // streamed generic variant
    out[0] = 7; out[1] = 0; out[2] = 1; out[3] = 0;
    return TP_OK;
  }
  if (st != TP_OK) return st;
  out[0] = pl.variant; out[1] = pl.P;
  out[2] = (pl.variant == 1 || pl.variant == 3) ? pl.a.Pq : (pl.variant == 8 ? pl.rows.a.S : (pl.variant == 9 ? 1 + pl.w.a.pair : 1));
  out[3] = (int)pl.smem;
  return TP_OK;
}

size_t tp_cp_als_ws_bytes(int d, const int* q, int R, int r, int grid) {
  AlsPlan pl;
  const int st = g_variant == 7 ? TP_EUNSUPPORTED : plan_als(d, q, R, r, grid, pl);
  if (st == TP_EUNSUPPORTED) return als_generic_ws_bytes(d, q, R, r);
  if (st != TP_OK) return 0;
  return pl.ws_total;
}

int tp_cp_als_f64(int d, const int* q, int R, const double* V, int r, double* U,
                  int sweeps, double reg, int reg_mode, double tol, double stall,
                  double* trace, int* info, int grid, void* ws, size_t ws_bytes, void* stream) {
  if (!V || !U || !info || sweeps < 0 || !(reg >= 0.0)) return TP_EINVAL;
  AlsPlan pl;
  int st = g_variant == 7 ? TP_EUNSUPPORTED : plan_als(d, q, R, r, grid, pl);
  if (st == TP_EUNSUPPORTED && als_generic_supported(d, q, R, r))
    return als_generic_run(d, q, R, V, r, U, sweeps, reg, reg_mode, tol, stall, trace, info, ws, ws_bytes,
                           (cudaStream_t)stream);
  if (st != TP_OK) return st;
  if (!ws || ws_bytes < pl.ws_total) return TP_EWORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (pl.variant == 9) {
    const int* redo = nullptr;
    const int pc = g_prof_cta < 0 ? pl.P + g_prof_cta : g_prof_cta;
    st = als_w_run(pl.w, V, U, sweeps, reg, reg_mode, tol, stall, trace, info, ws, align_up(pl.w.ws), s, g_prof, pc, &redo);
    if (st != TP_OK || sweeps == 0) return st;
    return als_rows_run(pl.rows, V, U, sweeps, reg, reg_mode, tol, stall, trace, info,
                        static_cast<char*>(ws) + align_up(pl.w.ws), ws_bytes - align_up(pl.w.ws), s, nullptr, 0,
                        g_ns_max > 0, redo);
  }
  if (pl.variant == 8)
    return als_rows_run(pl.rows, V, U, sweeps, reg, reg_mode, tol, stall, trace, info, ws, ws_bytes, s, g_prof,
                        g_prof_cta < 0 ? pl.P + g_prof_cta : g_prof_cta, g_ns_max > 0);
  AlsArgs& a = pl.a;
  Carver cv(ws, ws_bytes);
  a.G = cv.take<double>((size_t)d * r * r);
  a.Y = cv.take<double>(pl.ydoubles);
  a.ovl = cv.take<double>(pl.P);
  double* nsq = cv.take<double>(1);
  double* part = cv.take<double>(pl.ws_inner / sizeof(double));
  a.bar_ctr = cv.take<unsigned int>(16);
  a.Xprev = cv.take<double>(2 * (size_t)d * r * pad4(r));
  {
    long long nup = 0;
    for (int k = 0; k < d; ++k) nup += (long long)q[k] * pad4(r);
    a.Upad = cv.take<double>((size_t)nup);
  }
  a.ns_max = g_ns_max;
  a.V = V; a.U = U; a.trace = trace; a.info = info;
  a.sweeps = sweeps; a.reg = reg; a.reg_mode = reg_mode; a.tol = tol; a.stall = stall;
  a.need_resid = (trace != nullptr) || (tol > 0.0) || (stall > -INFINITY);
  a.norm_sq = nsq;
  a.prof = g_prof;
  a.prof_cta = g_prof_cta < 0 ? pl.P + g_prof_cta : g_prof_cta;
  a.dbg_skip = g_skip;
  cudaError_t e = cudaMemsetAsync(info, 0, 2 * sizeof(int), s);
  if (e != cudaSuccess) return cuda_status(e);
  e = cudaMemsetAsync(a.bar_ctr, 0, 16 * sizeof(unsigned int), s);
  if (e != cudaSuccess) return cuda_status(e);
  if (a.need_resid) {
    st = launch_inner(d, q, R, V, R, V, 1, nsq, part, s);   // ||V||^2 (cp.py:186-188)
    if (st != TP_OK) return st;
  }
  const void* fn = kernel_ptr(pl.rm, pl.variant, d);
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
  if (e != cudaSuccess) return cuda_status(e);
  if (pl.variant == 1 || pl.variant == 3) {
    if (pl.variant == 3 && pl.P > 8) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return cuda_status(e);
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = a.Pq; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.gridDim = dim3(pl.P); cfg.blockDim = dim3(ALS_NT); cfg.dynamicSmemBytes = pl.smem; cfg.stream = s;
    cfg.attrs = at; cfg.numAttrs = 2;
    // profiling aid: Nsight Compute cannot launch cooperative cluster kernels;
    // TP_ALS_NONCOOP=1 drops the cooperative attribute (co-residency then rests on
    // the occupancy check of plan_cluster, fine on an otherwise idle GPU)
    static const bool noncoop = getenv("TP_ALS_NONCOOP") && getenv("TP_ALS_NONCOOP")[0] == '1';
    // one cluster is co-scheduled by construction: no cooperative attribute (also
    // keeps the launch capturable in CUDA graphs)
    if (noncoop || pl.variant == 3) cfg.numAttrs = 1;
    void* args[] = {&a};
    e = cudaLaunchKernelExC(&cfg, fn, args);
    return cuda_status(e);
  }
  int per_sm = 0;
  const int nt = pl.variant == 5 ? TINY_NT : ((pl.variant == 2 && pl.rm == 8) ? ALS_SMALL_NT8 : ALS_NT);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, pl.smem);
  if (e != cudaSuccess) return cuda_status(e);
  if (per_sm < 1) return TP_EUNSUPPORTED;
  void* args[] = {&a};
  if (pl.P == 1)   // one CTA: a plain launch (graph-capturable; the grid barrier is a no-op)
    e = cudaLaunchKernel(fn, dim3(1), dim3(nt), args, pl.smem, s);
  else
    e = cudaLaunchCooperativeKernel(fn, dim3(pl.P), dim3(nt), args, pl.smem, s);
  return cuda_status(e);
}

// Fused operator apply + truncation for the one-CTA kernel: the target
// [A | scale * L(w)], w = [ws0 W0 | ws1 W1], is assembled inside als_tiny8 from the states
// and the operator's matrices (never written to global memory).  Fixed sweep count, no
// trace.  TP_EUNSUPPORTED when the plan is not the one-CTA kernel (the caller then
// materialises the target and calls tp_cp_als_f64).
int tp_cp_als_recipe_f64(int d, const int* q, int r, const double* A, int ra, const double* W0, double ws0,
                         const double* W1, double ws1, int rw, int n_terms, const double* w0, const int* mat_idx,
                         const double* mats, const long long* mat_off, int n_mats, double* U, int sweeps, double reg,
                         int reg_mode, int* info, void* ws, size_t ws_bytes, void* stream) {
  if (!A || !W0 || !U || !info || sweeps < 0 || !(reg >= 0.0) || ra < 1 || rw < 1 || n_terms < 1 || n_terms > 64 ||
      d < 1)
    return TP_EINVAL;
  if (d > TP_MAXD) return TP_EUNSUPPORTED;
  const int nw = W1 ? 2 : 1;
  const int R = ra + n_terms * nw * rw;
  AlsPlan pl;
  int st = plan_als(d, q, R, r, 0, pl);
  if (st != TP_OK) return st;
  if (pl.variant != 5) return TP_EUNSUPPORTED;
  if (!ws || ws_bytes < pl.ws_total) return TP_EWORKSPACE;
  std::vector<double> hw(w0, w0 + n_terms);
  std::vector<long long> hm((size_t)n_terms * d, -1);
  for (int t = 0; t < n_terms; ++t)
    for (int k = 0; k < d; ++k) {
      const int m = mat_idx[t * d + k];
      if (m >= 0) {
        if (m >= n_mats || !mats) return TP_EINVAL;
        hm[(size_t)t * d + k] = mat_off[m];
      }
    }
  const double* dw = device_table(hw);
  const long long* dm = device_table(hm);
  if (!dw || !dm) return TP_ECUDA;
  cudaStream_t s = (cudaStream_t)stream;
  AlsArgs& a = pl.a;
  Carver cv(ws, ws_bytes);
  a.G = cv.take<double>((size_t)d * r * r);
  a.Y = cv.take<double>(pl.ydoubles);
  a.ovl = cv.take<double>(pl.P);
  double* nsq = cv.take<double>(1);
  (void)cv.take<double>(pl.ws_inner / sizeof(double));
  a.bar_ctr = cv.take<unsigned int>(16);
  a.Xprev = cv.take<double>(2 * (size_t)d * r * pad4(r));
  a.ns_max = g_ns_max;
  a.V = nullptr; a.U = U; a.trace = nullptr; a.info = info;
  a.sweeps = sweeps; a.reg = reg; a.reg_mode = reg_mode; a.tol = 0.0; a.stall = -INFINITY;
  a.need_resid = 0;
  a.norm_sq = nsq;
  a.prof = g_prof; a.prof_cta = 0; a.dbg_skip = g_skip;
  a.rcp = 1; a.rcp_ra = ra; a.rcp_rw = rw; a.rcp_nw = nw; a.rcp_nt = n_terms;
  a.rcpA = A; a.rcpW[0] = W0; a.rcpW[1] = W1; a.rcp_ws[0] = ws0; a.rcp_ws[1] = ws1;
  a.rcp_w0 = dw; a.rcp_moff = dm; a.rcp_mats = mats;
  cudaError_t e = cudaMemsetAsync(info, 0, 2 * sizeof(int), s);
  if (e != cudaSuccess) return cuda_status(e);
  e = cudaFuncSetAttribute(tiny8_ptr(d), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
  if (e != cudaSuccess) return cuda_status(e);
  void* args[] = {&a};
  return cuda_status(cudaLaunchKernel(tiny8_ptr(d), dim3(1), dim3(TINY_NT), args, pl.smem, s));
}

}  // extern "C"

// ===========================================================================
// Input-rank-sharded ALS mode steps: a rank holds V[:, :, slab]
// (R_l columns) and the replicated guess U.  Per mode update j the host runs
//   tp_als_shard_rhs   (local partial of the right-hand side, r x Q_j)
//   allreduce           (NCCL over NVLink / gloo; sum over ranks)
//   tp_als_shard_update (A_j^-1, U_j, G_j, C_j[:, slab])
// which reproduces cp_approx_als (cp.py:310-320) up to summation order.
// ===========================================================================
#include "tp_gemm.cuh"

namespace tp {

struct ShardDims {
  int d, Rl, r, qmax;
  int q[TP_MAXD];
  long long offV[TP_MAXD], offU[TP_MAXD];
};

static int shard_dims(int d, const int* q, int Rl, int r, ShardDims& s) {
  if (d < 1 || d > TP_MAXD || Rl < 1 || r < 1 || r > 32 || !q) return TP_EINVAL;
  memset(&s, 0, sizeof(s));
  s.d = d; s.Rl = Rl; s.r = r;
  long long ov = 0, ou = 0;
  for (int k = 0; k < d; ++k) {
    if (q[k] < 1) return TP_EINVAL;
    s.q[k] = q[k]; s.offV[k] = ov; s.offU[k] = ou;
    ov += (long long)q[k] * Rl; ou += (long long)q[k] * r;
    s.qmax = q[k] > s.qmax ? q[k] : s.qmax;
  }
  return TP_OK;
}

// hadT[c][l] = prod_{k != j} C_k[l][c]
__global__ void shard_had_kernel(int d, int r, int Rl, int j, const double* C, double* hadT) {
  const int n = r * Rl;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int c = e / r, l = e % r;
    double v = 1.0;
    for (int k = 0; k < d; ++k)
      if (k != j) v *= C[((size_t)k * r + l) * Rl + c];
    hadT[e] = v;
  }
}

// one CTA: A = prod_{k!=j} G_k + lambda I, inverse by the symmetric sweep
template <int RM>
__global__ void __launch_bounds__(ALS_NT) shard_inverse_kernel(int d, int r, int j, const double* G, double reg,
                                                               int reg_mode, double* Ainv, int* info) {
  extern __shared__ double ss[];
  AlsArgs a;
  memset(&a, 0, sizeof(a));
  a.d = d; a.r = r; a.reg = reg; a.reg_mode = reg_mode;
  Smem sm;
  memset(&sm, 0, sizeof(sm));
  sm.Gs = ss;
  sm.pub = sm.Gs + (size_t)d * r * r;
  sm.part = sm.pub + 72;
  for (int e = threadIdx.x; e < d * r * r; e += ALS_NT) sm.Gs[e] = G[e];
  __syncthreads();
  const int bad = gram_inverse<RM>(a, sm, j, Ainv, r + 1);
  if (bad && threadIdx.x == 0) atomicOr(info, 1);
}

static cudaError_t gemm(int M, int N, int K, const double* A, long long sAm, long long sAk, const double* B,
                        long long sBk, long long sBn, double* C, long long sCm, long long sCn, cudaStream_t st) {
  return bgemm_launch(bgemm_desc(M, N, K, A, sAm, sAk, B, sBk, sBn, C, sCm, sCn), st);
}

}  // namespace tp

extern "C" {

size_t tp_als_shard_ws_bytes(int d, const int* q, int Rl, int r) {
  ShardDims s;
  if (shard_dims(d, q, Rl, r, s) != TP_OK) return 0;
  return align_up(8 * (size_t)r * Rl) + align_up(8 * (size_t)r * (r + 1)) + 256;
}

int tp_als_shard_init_f64(int d, const int* q, int Rl, const double* V, int r, const double* U, double* C,
                          double* G, void* stream) {
  ShardDims s;
  int st = shard_dims(d, q, Rl, r, s);
  if (st != TP_OK) return st;
  if (!V || !U || !C || !G) return TP_EINVAL;
  cudaStream_t cs = (cudaStream_t)stream;
  for (int k = 0; k < d; ++k) {
    const double* Uk = U + s.offU[k];
    cudaError_t e = gemm(r, Rl, s.q[k], Uk, 1, r, V + s.offV[k], Rl, 1, C + (size_t)k * r * Rl, Rl, 1, cs);
    if (e == cudaSuccess) e = gemm(r, r, s.q[k], Uk, 1, r, Uk, r, 1, G + (size_t)k * r * r, r, 1, cs);
    if (e != cudaSuccess) return cuda_status(e);
  }
  return TP_OK;
}

int tp_als_shard_rhs_f64(int d, const int* q, int Rl, const double* V, int r, const double* C, int j,
                         double* rhs, void* ws, size_t ws_bytes, void* stream) {
  ShardDims s;
  int st = shard_dims(d, q, Rl, r, s);
  if (st != TP_OK) return st;
  if (!V || !C || !rhs || j < 0 || j >= d) return TP_EINVAL;
  if (!ws || ws_bytes < tp_als_shard_ws_bytes(d, q, Rl, r)) return TP_EWORKSPACE;
  cudaStream_t cs = (cudaStream_t)stream;
  double* hadT = static_cast<double*>(ws);
  shard_had_kernel<<<(r * Rl + 255) / 256, 256, 0, cs>>>(d, r, Rl, j, C, hadT);
  // rhs[l][s] = sum_c had[l][c] V_j[s][c]      (cp.py:197-203)
  cudaError_t e = gemm(r, s.q[j], Rl, hadT, 1, r, V + s.offV[j], 1, Rl, rhs, s.q[j], 1, cs);
  return cuda_status(e == cudaSuccess ? cudaGetLastError() : e);
}

int tp_als_shard_update_f64(int d, const int* q, int Rl, const double* V, int r, double* U, double* C, double* G,
                            int j, const double* rhs, double reg, int reg_mode, int* info, void* ws,
                            size_t ws_bytes, void* stream) {
  ShardDims s;
  int st = shard_dims(d, q, Rl, r, s);
  if (st != TP_OK) return st;
  if (!V || !U || !C || !G || !rhs || !info || j < 0 || j >= d || !(reg >= 0.0)) return TP_EINVAL;
  if (!ws || ws_bytes < tp_als_shard_ws_bytes(d, q, Rl, r)) return TP_EWORKSPACE;
  cudaStream_t cs = (cudaStream_t)stream;
  double* Ainv = static_cast<double*>(ws) + align_up(8 * (size_t)r * Rl) / 8;
  const int rm = r <= 8 ? 8 : (r <= 16 ? 16 : 32);
  const size_t smem = sizeof(double) * ((size_t)d * r * r + 72 + ALS_PART);
  const void* fn = rm == 8 ? (const void*)shard_inverse_kernel<8>
                           : (rm == 16 ? (const void*)shard_inverse_kernel<16> : (const void*)shard_inverse_kernel<32>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (rm == 8) shard_inverse_kernel<8><<<1, ALS_NT, smem, cs>>>(d, r, j, G, reg, reg_mode, Ainv, info);
  else if (rm == 16) shard_inverse_kernel<16><<<1, ALS_NT, smem, cs>>>(d, r, j, G, reg, reg_mode, Ainv, info);
  else shard_inverse_kernel<32><<<1, ALS_NT, smem, cs>>>(d, r, j, G, reg, reg_mode, Ainv, info);
  cudaError_t e = cudaGetLastError();
  double* Uj = U + s.offU[j];
  const int Q = s.q[j], rp = r + 1;
  // U_j[s][i] = sum_m Ainv[i][m] rhs[m][s]       (cp.py:317)
  if (e == cudaSuccess) e = gemm(Q, r, r, rhs, 1, Q, Ainv, 1, rp, Uj, r, 1, cs);
  // G_j = U_j^T U_j, C_j[:, slab] = U_j^T V_j[:, slab]   (cp.py:318-320)
  if (e == cudaSuccess) e = gemm(r, r, Q, Uj, 1, r, Uj, r, 1, G + (size_t)j * r * r, r, 1, cs);
  if (e == cudaSuccess) e = gemm(r, Rl, Q, Uj, 1, r, V + s.offV[j], Rl, 1, C + (size_t)j * r * Rl, Rl, 1, cs);
  return cuda_status(e);
}

}  // extern "C"

// ===========================================================================
// Host side of the R-sharded fused truncation (als_xg).
// ===========================================================================
namespace tp {

struct XgPlan {
  AlsPlan pl;
  int Pg = 0, Pr = 0, PrT = 0, CH = 1;
  long long yhalf = 0;
  size_t ws_group = 0, peer_bytes = 0;
};

static const void* xg_kernel_ptr(int rm) {
  switch (rm) {
    case 8: return (const void*)als_xg<8>;
    case 16: return (const void*)als_xg<16>;
    default: return (const void*)als_xg<32>;
  }
}

// Pq = 4 CTAs per cluster (the single-GPU plan's choice for config 1); Pr clusters per
// rank such that all ngroups x Pr clusters are co-resident and the rank-major
// staging of ngpu x Pr partial slices fits; total clusters capped at 32 (the
// single-GPU optimum), equal R-slabs preferred.
static int plan_xg(int d, const int* q, int Rl, int r, int ngpu, int ngroups, XgPlan& xp) {
  if (d < 1 || d > TP_MAXD || Rl < 1 || r < 1 || !q || ngpu < 1 || ngpu > TP_MAXG || ngroups < 1 ||
      ngroups > ngpu)
    return TP_EINVAL;
  for (int k = 0; k < d; ++k) if (q[k] < 1) return TP_EINVAL;
  AlsPlan& pl = xp.pl;
  pl.rm = choose_rm(r);
  if (!pl.rm || (r & 1)) return TP_EUNSUPPORTED;
  int dev = 0, nsm = 148, smem_optin = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  } else {
    cudaGetLastError();
  }
  if (smem_optin <= 0) smem_optin = 227 * 1024;
  memset(&pl.a, 0, sizeof(pl.a));
  AlsArgs& a = pl.a;
  int qmin = q[0], qmax = 0;
  long long ov = 0, ou = 0, oup = 0;
  for (int k = 0; k < d; ++k) {
    qmin = q[k] < qmin ? q[k] : qmin;
    qmax = q[k] > qmax ? q[k] : qmax;
    a.q[k] = q[k]; a.qs[k] = pad4(q[k]); a.offV[k] = ov; a.offU[k] = ou; a.offUp[k] = oup;
    ov += (long long)q[k] * Rl; ou += (long long)q[k] * r; oup += (long long)q[k] * pad4(r);
  }
  a.d = d; a.R = Rl; a.r = r; a.qmax = qmax;
  const int Pq = 4;
  if (Pq > qmin) return TP_EUNSUPPORTED;
  const void* fn = xg_kernel_ptr(pl.rm);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  cudaGetLastError();
  auto try_pr = [&](int Pr) -> bool {
    const int P = Pr * Pq, PrT = Pr * ngpu, wmax = (Rl + Pr - 1) / Pr, ldw = pad4(wmax);
    const int ncolmax = (qmax + P - 1) / P;
    int sumnb = 0, nbmax = 0;
    for (int k = 0; k < d; ++k) {
      const int nb = (q[k] + Pq - 1) / Pq;
      sumnb += (nb + 3) & ~3;
      nbmax = nb > nbmax ? nb : nbmax;
    }
    sumnb += 8;
    const int mtr = (r + 7) / 8, nG = mtr * (mtr + 1) / 2;
    int chunk = r * wmax + ((nG + Pr - 1) / Pr) * 64;
    chunk += chunk & 1;
    // chunk slots: as many slices as fit twice into the U block staging (no extra smem)
    const size_t ust = (size_t)(((nbmax + 3) & ~3) + 1) * pad4(r), nbk = (size_t)ncolmax * r;
    int CH = (int)(ust / (2 * nbk));
    if (CH < 1) CH = 1;
    if (CH > Pr) CH = Pr;
    const size_t smem = cl_smem_doubles(d, r, wmax, ldw, sumnb, nbmax, ncolmax, 2 * CH, Pq, chunk, qmax) * sizeof(double);
    if (smem > (size_t)smem_optin) return false;
    (void)PrT;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = Pq; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(P * ngroups); cfg.blockDim = dim3(ALS_NT); cfg.dynamicSmemBytes = smem;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nclu = 0;
    if (cudaOccupancyMaxActiveClusters(&nclu, fn, &cfg) != cudaSuccess) { cudaGetLastError(); nclu = 0; }
    if (nclu < Pr * ngroups) return false;
    a.Pq = Pq; a.ldw = ldw; a.chunk = chunk; a.nbmax = nbmax; a.sumqs = sumnb;
    a.wmax = wmax; a.ncolmax = ncolmax; a.P = P;
    int qo = 0;
    for (int k = 0; k < d; ++k) { a.qoffc[k] = qo; qo += (((q[k] + Pq - 1) / Pq + 3) & ~3) * ldw; }
    pl.P = P; pl.Pr = Pr; pl.smem = smem; pl.variant = 6;
    xp.Pg = P; xp.Pr = Pr; xp.PrT = PrT; xp.CH = CH;
    xp.yhalf = (long long)P * Pr * ncolmax * r;
    xp.yhalf += xp.yhalf & 1;
    return true;
  };
  int Pr = nsm / (Pq * ngroups);
  if (Pr * ngpu > 32) Pr = 32 / ngpu > 0 ? 32 / ngpu : 1;
  if (Pr > Rl) Pr = Rl;
  bool ok = false;
  for (; Pr >= 1 && !ok; --Pr) {
    if (!try_pr(Pr)) continue;
    ok = true;
    const int wmax = (Rl + Pr - 1) / Pr;
    if (Rl % Pr != 0)
      for (int p2 = Pr - 1; p2 >= 1 && (Rl + p2 - 1) / p2 == wmax; --p2)
        if (Rl % p2 == 0) {
          if (!try_pr(p2)) try_pr(Pr);
          break;
        }
  }
  if (!ok) return TP_EUNSUPPORTED;
  long long nup = 0;
  for (int k = 0; k < d; ++k) nup += (long long)q[k] * pad4(r);
  xp.ws_group = align_up(sizeof(double) * (size_t)d * r * r) + align_up(16 * sizeof(unsigned int)) +
                align_up(sizeof(double) * 2 * (size_t)d * r * pad4(r)) + align_up(sizeof(double) * (size_t)nup) + 256;
  xp.peer_bytes = XG_HDR + 2 * (size_t)xp.yhalf * sizeof(double);
  a.ns_max = g_ns_max;
  return TP_OK;
}

}  // namespace tp

extern "C" {

size_t tp_als_xg_ws_bytes(int d, const int* q, int R_local, int r, int ngpu, int ngroups) {
  XgPlan xp;
  return plan_xg(d, q, R_local, r, ngpu, ngroups, xp) == TP_OK ? xp.ws_group : 0;
}

size_t tp_als_xg_peer_bytes(int d, const int* q, int R_local, int r, int ngpu, int ngroups) {
  XgPlan xp;
  return plan_xg(d, q, R_local, r, ngpu, ngroups, xp) == TP_OK ? xp.peer_bytes : 0;
}

int tp_als_xg_plan(int d, const int* q, int R_local, int r, int ngpu, int ngroups, int* out) {
  if (!out) return TP_EINVAL;
  XgPlan xp;
  const int st = plan_xg(d, q, R_local, r, ngpu, ngroups, xp);
  if (st != TP_OK) return st;
  out[0] = xp.Pg; out[1] = xp.pl.a.Pq; out[2] = xp.Pr; out[3] = (int)xp.pl.smem;
  return TP_OK;
}

int tp_als_xg_f64(int d, const int* q, int R_local, int r, int sweeps, double reg, int reg_mode,
                  int ngroups, const double* const* V, double* const* U, int* const* info,
                  void* const* ws, size_t ws_bytes, int ngpu, int rank0, void* const* peer, void* stream) {
  if (!V || !U || !info || !ws || !peer || sweeps < 0 || !(reg >= 0.0) || rank0 < 0 || rank0 + ngroups > ngpu)
    return TP_EINVAL;
  XgPlan xp;
  int st = plan_xg(d, q, R_local, r, ngpu, ngroups, xp);
  if (st != TP_OK) return st;
  if (ws_bytes < xp.ws_group) return TP_EWORKSPACE;
  for (int h = 0; h < ngpu; ++h) if (!peer[h]) return TP_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  AlsArgs a = xp.pl.a;
  a.sweeps = sweeps; a.reg = reg; a.reg_mode = reg_mode; a.tol = 0.0; a.stall = -INFINITY; a.need_resid = 0;
  XgArgs x;
  memset(&x, 0, sizeof(x));
  x.ngroups = ngroups; x.ngpu = ngpu; x.rank0 = rank0; x.Pg = xp.Pg; x.CH = xp.CH;
  x.yhalf = xp.yhalf;
  for (int h = 0; h < ngpu; ++h) x.peer[h] = static_cast<unsigned char*>(peer[h]);
  long long nup = 0;
  for (int k = 0; k < d; ++k) nup += (long long)q[k] * pad4(r);
  for (int g = 0; g < ngroups; ++g) {
    if (!V[g] || !U[g] || !info[g] || !ws[g]) return TP_EINVAL;
    Carver cv(ws[g], ws_bytes);
    XgGroup& gr = x.grp[g];
    gr.V = V[g]; gr.U = U[g]; gr.info = info[g];
    gr.G = cv.take<double>((size_t)d * r * r);
    gr.bar = cv.take<unsigned int>(16);
    gr.Xprev = cv.take<double>(2 * (size_t)d * r * pad4(r));
    gr.Upad = cv.take<double>((size_t)nup);
    cudaError_t e = cudaMemsetAsync(info[g], 0, 2 * sizeof(int), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(gr.bar, 0, 16 * sizeof(unsigned int), s);
    if (e != cudaSuccess) return cuda_status(e);
  }
  const void* fn = xg_kernel_ptr(xp.pl.rm);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xp.pl.smem);
  if (e != cudaSuccess) return cuda_status(e);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.Pq; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.gridDim = dim3(xp.Pg * ngroups); cfg.blockDim = dim3(ALS_NT); cfg.dynamicSmemBytes = xp.pl.smem; cfg.stream = s;
  cfg.attrs = at; cfg.numAttrs = 2;
  void* args[] = {&a, &x};
  e = cudaLaunchKernelExC(&cfg, fn, args);
  return cuda_status(e);
}

int tp_dev_alloc(size_t bytes, void** ptr) {
  if (!ptr || bytes == 0) return TP_EINVAL;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, bytes);
  return cuda_status(e);
}

int tp_dev_free(void* ptr) { return cuda_status(cudaFree(ptr)); }

int tp_ipc_handle(void* ptr, void* handle) {
  if (!ptr || !handle) return TP_EINVAL;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e == cudaSuccess) memcpy(handle, &h, sizeof(h));
  return cuda_status(e);
}

int tp_ipc_open(const void* handle, void** ptr) {
  if (!ptr || !handle) return TP_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
}

int tp_ipc_close(void* ptr) { return cuda_status(cudaIpcCloseMemHandle(ptr)); }

}  // extern "C"
