// Batched hierarchical-Tucker truncation by hSVD (ht.truncate, ht.py:313-372)
// for sm_100a.
//
// Same truncation as the reference, computed in the Gramian gauge instead of
// an explicit QR orthogonalization (ht.py:294-310):
//   1. frame Grams, leaves -> root:  M_leaf = U^T U,  M_t = B_t^T (M_l (x) M_r) B_t
//      (the root's 1x1 frame Gram is ||h||^2, ht.py:279-282);
//   2. environment Grams in the original gauge, root -> leaves:
//      Gh_l = sum B Gh_t M_r B^T,  Gh_r = sum B Gh_t M_l B^T;
//   3. per non-root node: M_t = V L V^T (Jacobi), node Gram in the orthonormal
//      gauge G_t = L^1/2 V^T Gh_t V L^1/2 (== the reference's node Gram up to an
//      orthogonal change of basis, so the spectrum and the keep rule
//      ht.py:346-359 are identical), G_t = W S W^T (Jacobi, descending);
//   4. S_t = V L^+1/2 W[:, :keep] maps the old frame to the kept orthonormal
//      one; projection U' = U S (leaves), B' = (S_l^T M_l (x) S_r^T M_r) B_t S_t
//      (interior, ht.py:361-370).
// Every contraction is a batched strided DMMA GEMM (tp_gemm.cuh); the batch runs
// over tensors x tree nodes of one level wave.
#include "tp_common.cuh"
#include "tp_gemm.cuh"
#include <cstring>
#include <vector>

namespace tp {

cudaError_t launch_tridiag_eigh(int nmat, int k, int nn, int first, int per, const double* Ain, double* Vout,
                                double* wout, int nvec, const int* skip, cudaStream_t st);

struct Tree {
  int n = 0, nleaf = 0, nint = 0, H = 0;
  int parent[32], left[32], right[32], slot[32], height[32], depth[32], dims[32];
};

static int build_tree(Tree& T, int lo, int hi, int par, int dep) {
  const int idx = T.n++;
  T.parent[idx] = par;
  T.depth[idx] = dep;
  T.dims[idx] = hi - lo;
  if (hi - lo == 1) {
    T.left[idx] = T.right[idx] = -1;
    T.slot[idx] = T.nleaf++;
    T.height[idx] = 0;
  } else {
    T.slot[idx] = T.nint++;
    const int half = (hi - lo) / 2;                 // left child takes the floor (ht.py:91)
    T.left[idx] = build_tree(T, lo, lo + half, idx, dep + 1);
    T.right[idx] = build_tree(T, lo + half, hi, idx, dep + 1);
    const int h = 1 + (T.height[T.left[idx]] > T.height[T.right[idx]] ? T.height[T.left[idx]] : T.height[T.right[idx]]);
    T.height[idx] = h;
  }
  if (T.height[idx] > T.H) T.H = T.height[idx];
  return idx;
}

// ---------------------------------------------------------------------------
// Batched cyclic Jacobi eigensolver for symmetric k x k matrices (k <= 64).
// Round-robin (circle-method) ordering: each round rotates k/2 disjoint pairs
// in parallel; rows, then columns and eigenvectors, are updated by all 256
// threads.  Output: eigenvalues descending, eigenvectors as columns.
// Matrix z lives at base index (z / per) * nn + first + z % per.
// ---------------------------------------------------------------------------
constexpr int JAC_NT = 256;

__global__ void __launch_bounds__(JAC_NT) jacobi_eigh_kernel(int k, int nn, int first, int per, const double* Ain,
                                                             double* Vout, double* wout, int max_sweeps, double tol,
                                                             int* sweeps_out, const int* skip) {
  extern __shared__ double js[];
  const int kp = k + (k & 1), ld = kp + 1;
  double* a = js;
  double* v = a + (size_t)kp * ld;
  double* cs = v + (size_t)kp * ld;          // [kp/2][2]
  int* pq = reinterpret_cast<int*>(cs + kp);  // [kp/2][2]
  double* red = cs + 2 * kp;                  // [JAC_NT]
  const int z = blockIdx.x;
  const size_t base = (size_t)(z / per) * nn + first + z % per;
  if (skip && skip[base]) return;   // factor already available (Cholesky)
  const double* in = Ain + base * k * k;
  const int tid = threadIdx.x;
  for (int e = tid; e < kp * kp; e += JAC_NT) {
    const int i = e / kp, j = e % kp;
    double x = 0.0;
    if (i < k && j < k) x = 0.5 * (in[i * k + j] + in[j * k + i]);   // eigh(0.5 (G + G^T)), ht.py:347
    a[i * ld + j] = x;
    v[i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int half = kp / 2, lane = tid & 31, warp = tid >> 5;
  // work split: warp w owns pairs w, w + 8, ...; its lanes run along the
  // contiguous row / the column (conflict-free shared accesses, warp-uniform skips)
  int* flag = reinterpret_cast<int*>(red);
  int sw = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    sw = sweep + 1;
    if (tid == 0) flag[0] = 0;
    __syncthreads();
    for (int round = 0; round < kp - 1; ++round) {
      if (tid < half) {
        const int m1 = kp - 1;
        int p = round, q = m1;
        if (tid != 0) {
          p = round + tid; p -= (p >= m1) ? m1 : 0;
          q = round - tid; q += (q < 0) ? m1 : 0;
        }
        if (p > q) { const int t = p; p = q; q = t; }
        const double apq = a[p * ld + q], app = a[p * ld + p], aqq = a[q * ld + q];
        double c = 1.0, s = 0.0;
        // threshold Jacobi: rotate only if a_pq is not negligible against the
        // diagonal (relative accuracy criterion) -- a sweep without rotations
        // means convergence.  Rotation from MUFU seeds + Newton steps.
        if (fabs(apq) > 1e-300 && apq * apq > (tol * tol) * fabs(app * aqq)) {
          const double tau = (aqq - app) * rcp_nr(2.0 * apq), at = fabs(tau);
          double t;
          if (at < 1e100) {
            const double h = fma(tau, tau, 1.0);
            t = (tau >= 0.0 ? 1.0 : -1.0) * rcp_nr(at + h * rsqrt_nr(h));
          } else {
            t = (tau >= 0.0 ? 0.5 : -0.5) * rcp_nr(at);
          }
          c = rsqrt_nr(fma(t, t, 1.0));
          s = t * c;
          flag[0] = 1;
        }
        cs[2 * tid] = c; cs[2 * tid + 1] = s;
        pq[2 * tid] = p; pq[2 * tid + 1] = q;
      }
      __syncthreads();
      for (int pr = warp; pr < half; pr += JAC_NT / 32) {     // rows p, q
        const double s = cs[2 * pr + 1];
        if (s == 0.0) continue;
        const int p = pq[2 * pr], q = pq[2 * pr + 1];
        const double c = cs[2 * pr];
        for (int j = lane; j < kp; j += 32) {
          const double x = a[p * ld + j], y = a[q * ld + j];
          a[p * ld + j] = c * x - s * y;
          a[q * ld + j] = s * x + c * y;
        }
      }
      __syncthreads();
      for (int pr = warp; pr < half; pr += JAC_NT / 32) {     // columns p, q and eigenvectors
        const double s = cs[2 * pr + 1];
        if (s == 0.0) continue;
        const int p = pq[2 * pr], q = pq[2 * pr + 1];
        const double c = cs[2 * pr];
        for (int i = lane; i < kp; i += 32) {
          const double x = a[i * ld + p], y = a[i * ld + q];
          a[i * ld + p] = c * x - s * y;
          a[i * ld + q] = s * x + c * y;
          const double vx = v[i * ld + p], vy = v[i * ld + q];
          v[i * ld + p] = c * vx - s * vy;
          v[i * ld + q] = s * vx + c * vy;
        }
      }
      __syncthreads();
    }
    if (flag[0] == 0) break;
    __syncthreads();
  }
  if (sweeps_out && tid == 0) atomicAdd(sweeps_out, sw);
  // sort descending (ties by index), write eigenvalues and eigenvector columns
  double* Vo = Vout + base * k * k;
  double* wo = wout + base * k;
  int* rank = pq;   // reuse (kp/2*2 >= k ints)
  __syncthreads();
  if (tid < k) {
    const double wi = a[tid * ld + tid];
    int rk = 0;
    for (int j = 0; j < k; ++j) {
      const double wj = a[j * ld + j];
      if (wj > wi || (wj == wi && j < tid)) ++rk;
    }
    rank[tid] = rk;
    wo[rk] = wi;
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += JAC_NT) {
    const int i = e / k, m = e % k;
    Vo[i * k + rank[m]] = v[i * ld + m];
  }
}

// Same cyclic Jacobi (identical pair ordering, rotation formula and threshold),
// one barrier per round instead of three: every warp recomputes the k/2
// rotations of the round (lane = pair, warp-uniform results, no shared
// hand-off), and the two-sided update A <- J^T A J is done as independent 2x2
// blocks (rows of pair P, columns of pair P'), read from one buffer and written
// to the other (double-buffered A, so angle reads and block writes of a round
// never race).  Eigenvector columns are rotated in place by their owner lane.
// Warp w owns row pairs w, w + 8, w + 16, w + 24; lane l owns column pair l.
__global__ void __launch_bounds__(JAC_NT) jacobi_db_kernel(int k, int nn, int first, int per, const double* Ain,
                                                           double* Vout, double* wout, int max_sweeps, double tol,
                                                           int* sweeps_out, const int* skip) {
  extern __shared__ double js[];
  const int kp = k + (k & 1), ld = kp + 1, half = kp / 2, m1 = kp - 1;
  double* Ac = js;
  double* An = Ac + (size_t)kp * ld;
  double* v = An + (size_t)kp * ld;
  const int z = blockIdx.x;
  const size_t base = (size_t)(z / per) * nn + first + z % per;
  if (skip && skip[base]) return;
  const double* in = Ain + base * k * k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < kp * kp; e += JAC_NT) {
    const int i = e / kp, j = e % kp;
    double x = 0.0;
    if (i < k && j < k) x = 0.5 * (in[i * k + j] + in[j * k + i]);   // eigh(0.5 (G + G^T)), ht.py:347
    Ac[i * ld + j] = x;
    v[i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const bool live = lane < half;
  const double tol2 = tol * tol;
  int sw = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    sw = sweep + 1;
    bool any = false;
    for (int round = 0; round < m1; ++round) {
      int p = round, q = m1;
      if (lane != 0) {   // (round + lane) mod m1, (round - lane) mod m1 without integer division
        p = round + lane; p -= (p >= m1) ? m1 : 0;
        q = round - lane; q += (q < 0) ? m1 : 0;
      }
      if (p > q) { const int t = p; p = q; q = t; }
      double c = 1.0, s = 0.0, t = 0.0;
      int rot = 0;
      if (live) {
        const double apq = Ac[p * ld + q], app = Ac[p * ld + p], aqq = Ac[q * ld + q];
        // |a_pq| > tol sqrt(|a_pp a_qq|) without the square root; rotation from
        // MUFU seeds refined by Newton steps (no IEEE div / sqrt sequences)
        if (fabs(apq) > 1e-300 && apq * apq > tol2 * fabs(app * aqq)) {
          const double tau = (aqq - app) * rcp_nr(2.0 * apq), at = fabs(tau);
          if (at < 1e100) {
            const double h = fma(tau, tau, 1.0);
            const double sq = h * rsqrt_nr(h);                     // sqrt(1 + tau^2)
            t = (tau >= 0.0 ? 1.0 : -1.0) * rcp_nr(at + sq);
          } else {
            t = (tau >= 0.0 ? 0.5 : -0.5) * rcp_nr(at);            // 1 / (2 tau): tau^2 would overflow
          }
          c = rsqrt_nr(fma(t, t, 1.0));
          s = t * c;
          rot = 1;
        }
      }
      any |= __any_sync(0xffffffffu, rot) != 0;
      // eigenvector columns p, q (rows warp, warp + 8, ...)
      if (live && rot) {
        for (int i = warp; i < kp; i += JAC_NT / 32) {
          const double vx = v[i * ld + p], vy = v[i * ld + q];
          v[i * ld + p] = c * vx - s * vy;
          v[i * ld + q] = s * vx + c * vy;
        }
      }
      double apq_d = 0.0;
      if (live) apq_d = Ac[p * ld + q];
      for (int P = warp; P < half; P += JAC_NT / 32) {
        const int pP = __shfl_sync(0xffffffffu, p, P), qP = __shfl_sync(0xffffffffu, q, P);
        const double cP = __shfl_sync(0xffffffffu, c, P), sP = __shfl_sync(0xffffffffu, s, P);
        if (!live) continue;
        double* r0 = An + pP * ld;
        double* r1 = An + qP * ld;
        if (P == lane) {        // diagonal block: the rotation annihilates a_pq exactly
          if (rot) {
            r0[pP] = Ac[pP * ld + pP] - t * apq_d;
            r1[qP] = Ac[qP * ld + qP] + t * apq_d;
            r0[qP] = 0.0;
            r1[pP] = 0.0;
          } else {
            r0[pP] = Ac[pP * ld + pP]; r0[qP] = Ac[pP * ld + qP];
            r1[pP] = Ac[qP * ld + pP]; r1[qP] = Ac[qP * ld + qP];
          }
          continue;
        }
        const double x00 = Ac[pP * ld + p], x01 = Ac[pP * ld + q];
        const double x10 = Ac[qP * ld + p], x11 = Ac[qP * ld + q];
        const double y00 = cP * x00 - sP * x10, y01 = cP * x01 - sP * x11;   // rows (pair P)
        const double y10 = sP * x00 + cP * x10, y11 = sP * x01 + cP * x11;
        r0[p] = c * y00 - s * y01; r0[q] = s * y00 + c * y01;                // columns (pair P')
        r1[p] = c * y10 - s * y11; r1[q] = s * y10 + c * y11;
      }
      __syncthreads();
      double* tmp = Ac; Ac = An; An = tmp;
    }
    if (!any) break;
  }
  if (sweeps_out && tid == 0) atomicAdd(sweeps_out, sw);
  double* Vo = Vout + base * k * k;
  double* wo = wout + base * k;
  int* rank = reinterpret_cast<int*>(An);   // scratch (An is dead after the last barrier)
  if (tid < k) {
    const double wi = Ac[tid * ld + tid];
    int rk = 0;
    for (int j = 0; j < k; ++j) {
      const double wj = Ac[j * ld + j];
      if (wj > wi || (wj == wi && j < tid)) ++rk;
    }
    rank[tid] = rk;
    wo[rk] = wi;
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += JAC_NT) {
    const int i = e / k, m = e % k;
    Vo[i * k + rank[m]] = v[i * ld + m];
  }
}

// Same cyclic Jacobi (pair ordering, rotation formula, threshold) on the upper
// triangle only, as independent 2x2 blocks: per round, warp 0 computes the k/2
// rotations (and updates the diagonal blocks) while warps 1.. apply the PREVIOUS
// round's rotations to the eigenvector columns; one barrier; then every thread
// updates ~2 of the (k/2)(k/2-1)/2 off-diagonal upper blocks (rows of pair P,
// columns of pair P' > P) in place; one barrier.  Half the shared traffic and ~1/4 of the instructions of the
// row-then-column kernel.  Matrix z lives at base index (z / per) * nn + first + z % per.
__global__ void __launch_bounds__(JAC_NT) jacobi_sym_kernel(int k, int nn, int first, int per, const double* Ain,
                                                            double* Vout, double* wout, int max_sweeps, double tol,
                                                            int* sweeps_out, const int* skip) {
  extern __shared__ double js[];
  const int kp = k + (k & 1), ld = kp + 1, half = kp / 2, m1 = kp - 1;
#define PK(i, j) ((i) * kp - (((i) * ((i) + 1)) >> 1) + (j))   // packed upper index, i <= j
  double* a = js;                              // packed upper triangle: (i <= j) at a[PK(i, j)]
  double* v = a + (size_t)kp * (kp + 1) / 2;   // [kp][ld]
  double* rot = v + (size_t)kp * ld;           // [2][32][3]: c, s, t (round parity)
  int* rpq = reinterpret_cast<int*>(rot + 2 * 32 * 3);   // [2][32][2]: p, q
  int* flagbuf = rpq + 2 * 32 * 2;             // [2] per sweep parity
  unsigned short* blk = reinterpret_cast<unsigned short*>(flagbuf + 2);   // [nblk]: P | P' << 8
  const int z = blockIdx.x;
  const size_t base = (size_t)(z / per) * nn + first + z % per;
  if (skip && skip[base]) return;
  const double* in = Ain + base * k * k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < kp * kp; e += JAC_NT) {
    const int i = e / kp, j = e % kp;
    double x = 0.0;
    if (i < k && j < k) x = 0.5 * (in[i * k + j] + in[j * k + i]);   // eigh(0.5 (G + G^T)), ht.py:347
    if (i <= j) a[PK(i, j)] = x;
    v[i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  const int nblk = half * (half - 1) / 2;   // off-diagonal upper blocks (diagonal ones: warp 0)
  for (int b = tid; b < nblk; b += JAC_NT) {
    int P = 0, rem = b;
    while (rem >= half - 1 - P) { rem -= half - 1 - P; ++P; }
    blk[b] = (unsigned short)(P | ((P + 1 + rem) << 8));
  }
  __syncthreads();
  const double tol2 = tol * tol;
  bool any = false;    // warp 0: rotations in this sweep
  int sw = 0, pending = -1, gr = 0;   // pending: round parity whose rotations still await the eigenvector update
  // eigenvector columns p, q of each rotated pair: warp per pair (uniform skip and
  // parameter loads), lanes along the rows
  auto v_update = [&](int par, int w0, int nw) {
    const double* R = rot + par * 96;
    const int* PQ = rpq + par * 64;
    for (int P = warp - w0; P < half; P += nw) {
      const double s_ = R[3 * P + 1];
      if (s_ == 0.0) continue;
      const double c_ = R[3 * P];
      const int p = PQ[2 * P], q = PQ[2 * P + 1];
      for (int i = lane; i < kp; i += 32) {
        const double vx = v[i * ld + p], vy = v[i * ld + q];
        v[i * ld + p] = c_ * vx - s_ * vy;
        v[i * ld + q] = s_ * vx + c_ * vy;
      }
    }
  };
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    sw = sweep + 1;
    any = false;
    for (int round = 0; round < m1; ++round, ++gr) {
      const int par = gr & 1;   // global round parity (m1 is odd: round parity would repeat across sweeps)
      if (warp == 0) {
        if (lane < half) {
          int p = round, q = m1;
          if (lane != 0) {
            p = round + lane; p -= (p >= m1) ? m1 : 0;
            q = round - lane; q += (q < 0) ? m1 : 0;
          }
          if (p > q) { const int t_ = p; p = q; q = t_; }
          const double apq = a[PK(p, q)], app = a[PK(p, p)], aqq = a[PK(q, q)];
          double c = 1.0, s_ = 0.0, t = 0.0;
          if (fabs(apq) > 1e-300 && apq * apq > tol2 * fabs(app * aqq)) {
            const double tau = (aqq - app) * rcp_nr(2.0 * apq), at = fabs(tau);
            if (at < 1e100) {
              const double h = fma(tau, tau, 1.0);
              t = (tau >= 0.0 ? 1.0 : -1.0) * rcp_nr(at + h * rsqrt_nr(h));
            } else {
              t = (tau >= 0.0 ? 0.5 : -0.5) * rcp_nr(at);
            }
            c = rsqrt_nr(fma(t, t, 1.0));
            s_ = t * c;
            any = true;
            // diagonal block of the pair (no other thread touches it this round)
            a[PK(p, p)] = app - t * apq;
            a[PK(q, q)] = aqq + t * apq;
            a[PK(p, q)] = 0.0;
          }
          double* R = rot + par * 96 + 3 * lane;
          R[0] = c; R[1] = s_; R[2] = t;
          rpq[par * 64 + 2 * lane] = p; rpq[par * 64 + 2 * lane + 1] = q;
        }
        if (round == m1 - 1) {
          const bool anyw = __any_sync(0xffffffffu, any);
          if (lane == 0) flagbuf[sweep & 1] = anyw ? 1 : 0;
        }
      } else if (pending >= 0) {
        v_update(pending, 1, JAC_NT / 32 - 1);
      }
      __syncthreads();
      // off-diagonal upper 2x2 blocks (rows of pair P, columns of pair P2 > P), in place
      const double* R = rot + par * 96;
      const int* PQ = rpq + par * 64;
      for (int b = tid; b < nblk; b += JAC_NT) {
        const int P = blk[b] & 0xff, P2 = blk[b] >> 8;
        const int p = PQ[2 * P], q = PQ[2 * P + 1];
        const double cP = R[3 * P], sP = R[3 * P + 1];
        const double c2 = R[3 * P2], s2 = R[3 * P2 + 1];
        if (sP == 0.0 && s2 == 0.0) continue;
        const int p2 = PQ[2 * P2], q2 = PQ[2 * P2 + 1];
        // storage of (row, col) in the upper triangle
        const int i00 = p < p2 ? PK(p, p2) : PK(p2, p);
        const int i01 = p < q2 ? PK(p, q2) : PK(q2, p);
        const int i10 = q < p2 ? PK(q, p2) : PK(p2, q);
        const int i11 = q < q2 ? PK(q, q2) : PK(q2, q);
        const double x00 = a[i00], x01 = a[i01], x10 = a[i10], x11 = a[i11];
        const double y00 = cP * x00 - sP * x10, y01 = cP * x01 - sP * x11;   // rows (pair P)
        const double y10 = sP * x00 + cP * x10, y11 = sP * x01 + cP * x11;
        a[i00] = c2 * y00 - s2 * y01; a[i01] = s2 * y00 + c2 * y01;          // columns (pair P2)
        a[i10] = c2 * y10 - s2 * y11; a[i11] = s2 * y10 + c2 * y11;
      }
      pending = par;
      __syncthreads();
    }
    if (flagbuf[sweep & 1] == 0) break;
  }
  if (pending >= 0) {
    v_update(pending, 0, JAC_NT / 32);
    __syncthreads();
  }
  if (sweeps_out && tid == 0) atomicAdd(sweeps_out, sw);
  double* Vo = Vout + base * k * k;
  double* wo = wout + base * k;
  int* rank = rpq;   // scratch
  if (tid < k) {
    const double wi = a[PK(tid, tid)];
    int rk = 0;
    for (int j = 0; j < k; ++j) {
      const double wj = a[PK(j, j)];
      if (wj > wi || (wj == wi && j < tid)) ++rk;
    }
    rank[tid] = rk;
    wo[rk] = wi;
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += JAC_NT) {
    const int i = e / k, m = e % k;
    Vo[i * k + rank[m]] = v[i * ld + m];
  }
#undef PK
}

// Frame-Gram square-root factor by Cholesky, M_t = L L^T (one CTA per non-root
// node, right-looking, 64 dependent steps instead of ~8 Jacobi sweeps).  In the
// Gramian gauge only a factor F with F F^T = M_t enters: with F = L instead of
// V diag(sqrt(l)) (ht.py:347-349) G_t = L^T Gh L has the same eigenvalues and
// S_t = L^-T W_keep is the same basis, so the truncation is unchanged.  Nodes whose
// Gram is numerically singular (a pivot <= 1e-12 max diag) keep the eigh path of
// the reference (pseudo-inverse square root): ok[node] = 0.
__global__ void __launch_bounds__(256) chol_frame_kernel(int k, int nn, const double* Mf, double* Lout, int* ok) {
  extern __shared__ double cs_[];
  const int z = blockIdx.x, per = nn - 1, ld = k + (((4 - k % 16) + 16) % 16), tid = threadIdx.x;
  const size_t base = (size_t)(z / per) * nn + 1 + z % per;
  double* A = cs_;
  double* dmax = A + (size_t)k * ld;
  const double* M = Mf + base * k * k;
  for (int e = tid; e < k * k; e += 256) {
    const int i = e / k, j = e - i * k;
    A[i * ld + j] = 0.5 * (M[e] + M[j * k + i]);
  }
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < k; ++i) m = fmax(m, A[i * ld + i]);
    dmax[0] = m;
    dmax[1] = 1.0;   // ok
  }
  __syncthreads();
  const double tol = 1e-12 * dmax[0];
  for (int j = 0; j < k; ++j) {
    const double piv = A[j * ld + j];
    if (!(piv > tol)) { if (tid == 0) dmax[1] = 0.0; break; }   // uniform: every thread reads the same piv
    const double dj = sqrt(piv), inv = 1.0 / dj;
    __syncthreads();
    for (int i = j + 1 + tid; i < k; i += 256) A[i * ld + j] *= inv;
    if (tid == 0) A[j * ld + j] = dj;
    __syncthreads();
    {   // trailing lower triangle (i >= c > j), 4 threads per row (no runtime divisions)
      const int row = tid >> 2, part = tid & 3;
      for (int i = j + 1 + row; i < k; i += 64) {
        const double aij = A[i * ld + j];
        for (int c = j + 1 + part; c <= i; c += 4) A[i * ld + c] = fma(-aij, A[c * ld + j], A[i * ld + c]);
      }
    }
    __syncthreads();
  }
  __syncthreads();
  const int good = dmax[1] != 0.0;
  if (tid == 0) ok[base] = good;
  if (!good) return;
  double* L = Lout + base * k * k;
  for (int e = tid; e < k * k; e += 256) {
    const int i = e / k, c = e - i * k;
    L[e] = (c <= i) ? A[i * ld + c] : 0.0;
  }
}

// G_t = diag(sqrt(l)) V^T Gh V diag(sqrt(l)) for every non-root node (one CTA each);
// nodes with a Cholesky factor (ok) use G_t = L^T Gh L
__global__ void __launch_bounds__(256) form_g_kernel(int k, int nn, const double* Vm, const double* lam,
                                                     const double* Gh, double* G, const int* ok, const int* bound) {
  extern __shared__ double fs[];
  const int z = blockIdx.x, per = nn - 1;
  const size_t base = (size_t)(z / per) * nn + 1 + z % per;
  const int ld = k + 1;
  double* V = fs;
  double* H = V + (size_t)k * ld;
  double* P = H + (size_t)k * ld;
  for (int e = threadIdx.x; e < k * k; e += 256) {
    const int i = e / k, j = e % k;
    V[i * ld + j] = Vm[base * k * k + e];
    H[i * ld + j] = Gh[base * k * k + e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += 256) {   // P = V^T H
    const int m = e / k, j = e % k;
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc = fma(V[i * ld + m], H[i * ld + j], acc);
    P[m * ld + j] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += 256) {   // G = P V, scaled
    const int m = e / k, n = e % k;
    double acc = 0.0;
    for (int j = 0; j < k; ++j) acc = fma(P[m * ld + j], V[j * ld + n], acc);
    if (ok[base]) { G[base * k * k + e] = acc; continue; }
    const int bt = bound[1 + z % per];
    const double sm = m < bt ? sqrt(fmax(lam[base * k + m], 0.0)) : 0.0;
    const double sn = n < bt ? sqrt(fmax(lam[base * k + n], 0.0)) : 0.0;
    G[base * k * k + e] = acc * sm * sn;
  }
}

// keep rule (ht.py:349-358) per (tensor, non-root node); discarded mass; ranks
// bound[t]: structural rank of node t (leaves min(Q, k), interior min(k, bound_l bound_r))
// -- the rank the reference's QR orthogonalisation (ht.py:294-310) leaves; eigenvalues
// past it are rounding noise of the Gramian gauge and are never kept
__global__ void keep_rule_kernel(int k, int nn, int nb, int ndim, double eps, int r_max, const double* sig,
                                 const double* Mf, int* keep, double* disc, const int* bound, double* Wz, int ro) {
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  const int per = nn - 1;
  if (z >= nb * per) return;
  const int b = z / per, t = 1 + z % per;
  const double total = sqrt(fmax(Mf[(size_t)b * nn * k * k], 0.0));
  const double budget = (eps * total) * (eps * total) / (double)(2 * ndim - 3 > 1 ? 2 * ndim - 3 : 1);
  const double* s = sig + ((size_t)b * nn + t) * k;
  int kp = k;
  double tail = 0.0;
  while (kp > 1) {
    const double step = fmax(s[kp - 1], 0.0);
    if (kp > r_max || kp > bound[nn + t] || tail + step <= budget) { tail += step; --kp; }
    else break;
  }
  keep[b * nn + t] = kp;
  disc[b * nn + t] = tail;
  if (Wz) {   // discarded eigenvectors -> zero columns (the GEMM formation of S_t / T_t)
    double* W = Wz + ((size_t)b * nn + t) * k * k;
    for (int i = 0; i < k; ++i)
      for (int c = kp; c < ro; ++c) W[(size_t)i * k + c] = 0.0;
  }
}

__global__ void finish_kernel(int k, int nn, int nb, const double* Mf, const int* keep, const double* disc,
                              double* est, double* norms, int* out_ranks) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  double s = 0.0;
  for (int t = 1; t < nn; ++t) s += disc[b * nn + t];
  est[b] = sqrt(fmax(s, 0.0));
  norms[b] = sqrt(fmax(Mf[(size_t)b * nn * k * k], 0.0));
  out_ranks[b * nn] = 1;
  for (int t = 1; t < nn; ++t) out_ranks[b * nn + t] = keep[b * nn + t];
}

// Frame factor F (M_t = F F^T on its range) and its pseudo-inverse Fi for every non-root
// node, so that the node Gram G_t = F^T Gh F and the kept basis S_t = Fi^T W_keep,
// T_t = W_keep^T F^T become batched DMMA GEMMs: Cholesky nodes F = L, Fi = L^-1 (column-
// parallel forward substitution, 4 threads per column); eigh nodes F = V diag(s),
// Fi = diag(mu) V^T with s = sqrt(l), mu = 1/sqrt(l) on the kept range (m < bound,
// l > 1e-14 l_max, the thresholded pseudo-inverse of form_st) and 0 elsewhere.
__global__ void __launch_bounds__(256) frame_factor_kernel(int k, int nn, const double* Vm, const double* lam,
                                                           const int* ok, const int* bound, double* Ff, double* Fi) {
  extern __shared__ double ffs[];
  const int z = blockIdx.x, per = nn - 1, tid = threadIdx.x;
  const size_t base = (size_t)(z / per) * nn + 1 + z % per;
  const double* V = Vm + base * k * k;
  double* F = Ff + base * k * k;
  double* X = Fi + base * k * k;
  if (!ok[base]) {
    const double lmax = fmax(lam[base * k], 0.0);
    const int bt = bound[1 + z % per];
    for (int e = tid; e < k * k; e += 256) {
      const int i = e / k, m = e - i * k;
      const double l = lam[base * k + m];
      const bool keep = m < bt && l > lmax * 1e-14 && l > 0.0;
      const double v = V[e];
      F[e] = keep ? v * sqrt(l) : 0.0;                   // F[i][m]
      X[(size_t)m * k + i] = keep ? v / sqrt(l) : 0.0;   // Fi[m][i]
    }
    return;
  }
  const int ld = k + 1;
  double* L = ffs;               // [k][k + 1]
  double* dinv = L + (size_t)k * ld;
  for (int e = tid; e < k * k; e += 256) {
    const int i = e / k, c = e - i * k;
    const double v = (c <= i) ? V[e] : 0.0;
    L[i * ld + c] = v;
    F[e] = v;
  }
  __syncthreads();
  for (int i = tid; i < k; i += 256) dinv[i] = 1.0 / L[i * ld + i];
  __syncthreads();
  // X = L^-1, column c by 4 threads: X[i][c] = (delta_ic - sum_{c<=m<i} L[i][m] X[m][c]) / L[i][i]
  double* Xs = dinv + k;         // [k][k + 1]
  for (int c0 = 0; c0 < k; c0 += 64) {
    const int c = c0 + (tid >> 2), part = tid & 3;
    for (int i = 0; i < k; ++i) {
      double acc = 0.0;
      if (c < k && i > c)
        for (int m = c + part; m < i; m += 4) acc = fma(L[i * ld + m], Xs[m * ld + c], acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (c < k && part == 0) Xs[i * ld + c] = (i < c) ? 0.0 : ((i == c ? 1.0 : 0.0) - acc) * dinv[i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += 256) X[e] = Xs[(e / k) * ld + e % k];
}

// S_t = V diag(l^+1/2) W[:, :keep] (k x ro, zero columns beyond keep); T_t = S_t^T M_t (ro x k)
__global__ void __launch_bounds__(256) form_st_kernel(int k, int ro, int nn, const double* Vm, const double* lam,
                                                      const double* Wg, const int* keep, const double* Mf,
                                                      double* S, double* T, const int* ok, const int* bound) {
  extern __shared__ double ss[];
  const int z = blockIdx.x, per = nn - 1;
  const size_t base = (size_t)(z / per) * nn + 1 + z % per;
  const int kp = keep[base];
  if (ok[base]) {
    // Cholesky factor: S = L^-T W_keep (back substitution, 16 threads per column),
    // T = S^T M = W_keep^T L^T
    // L, the kept columns of W and 1 / diag(L) staged in shared memory first (coalesced):
    // the 64-step back substitution then runs on shared operands only
    const double* L = Vm + base * k * k;
    const double* W = Wg + base * k * k;
    double* Sl = ss;                         // [k][ro]
    double* Ls = Sl + (size_t)k * ro;        // [k][k + 1]
    double* Ws = Ls + (size_t)k * (k + 1);   // [k][ro]
    double* dinv = Ws + (size_t)k * ro;      // [k]
    for (int e = threadIdx.x; e < k * k; e += 256) Ls[(e / k) * (k + 1) + e % k] = L[e];
    for (int e = threadIdx.x; e < k * ro; e += 256) Ws[e] = W[(e / ro) * k + e % ro];
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += 256) dinv[i] = 1.0 / Ls[i * (k + 1) + i];
    __syncthreads();
    // 16 columns per pass (16 threads per column); the passes are independent
    const int part = threadIdx.x & 15;
    for (int c0 = 0; c0 < ro; c0 += 16) {
      const int c = c0 + (threadIdx.x >> 4);
      for (int i = k - 1; i >= 0; --i) {
        double acc = 0.0;
        if (c < ro)
          for (int m = i + 1 + part; m < k; m += 16) acc = fma(Ls[m * (k + 1) + i], Sl[m * ro + c], acc);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (c < ro && part == 0) Sl[i * ro + c] = (c < kp) ? (Ws[i * ro + c] - acc) * dinv[i] : 0.0;
        __syncthreads();
      }
    }
    for (int e = threadIdx.x; e < k * ro; e += 256) S[base * k * ro + e] = Sl[e];
    for (int e = threadIdx.x; e < ro * k; e += 256) {
      const int cc = e / k, a2 = e % k;
      double acc = 0.0;
      if (cc < kp)
        for (int i = 0; i <= a2; ++i) acc = fma(Ws[i * ro + cc], Ls[a2 * (k + 1) + i], acc);
      T[base * ro * k + e] = acc;
    }
    return;
  }
  double* mu = ss;               // [k]
  double* Sl = mu + k;           // [k][ro]
  const double lmax = fmax(lam[base * k], 0.0);
  for (int m = threadIdx.x; m < k; m += 256) {
    const double l = lam[base * k + m];
    mu[m] = (m < bound[1 + z % per] && l > lmax * 1e-14 && l > 0.0) ? 1.0 / sqrt(l) : 0.0;
  }
  __syncthreads();
  const double* V = Vm + base * k * k;
  const double* W = Wg + base * k * k;
  for (int e = threadIdx.x; e < k * ro; e += 256) {
    const int i = e / ro, c = e % ro;
    double acc = 0.0;
    if (c < kp)
      for (int m = 0; m < k; ++m) acc = fma(V[i * k + m] * mu[m], W[m * k + c], acc);
    Sl[e] = acc;
    S[base * k * ro + e] = acc;
  }
  __syncthreads();
  const double* M = Mf + base * k * k;
  for (int e = threadIdx.x; e < ro * k; e += 256) {
    const int c = e / k, a2 = e % k;
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc = fma(Sl[i * ro + c], M[i * k + a2], acc);
    T[base * ro * k + e] = acc;
  }
}

// Bp[e][a][j] = B[a][e][j]  (k x k x kt per batch entry, offsets table)
__global__ void transpose12_kernel(int k, int kt, const long long* offs, const double* B, double* Bp, long long sBp) {
  const int z = blockIdx.y;
  const double* src = B + offs[3 * z];
  double* dst = Bp + z * sBp;
  const int n = k * k * kt;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int a = e / (k * kt), r = e % (k * kt), b = r / kt, j = r % kt;
    dst[(size_t)b * k * kt + a * kt + j] = src[e];
  }
}

__global__ void set_root_env(int k, int nn, int nb, double* Gh) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < nb) Gh[(size_t)b * nn * k * k] = 1.0;
}

// split-K partial tiles: bgemm_pick_split only splits below 2 x 148 x 2 CTAs of 64 x 64
constexpr size_t HT_PART = (size_t)GB_TM * GB_TN * 8 * 148;

struct HtPlan {
  Tree T;
  int d, Q, k, nb, ro, maxw;
  size_t big, off_n, total;
};

// any binary dimension tree (ht.py:55-76) given as parallel arrays, nodes[0] the
// root; leaf / interior slots in node order (the packed batch layout)
static int finish_tree(Tree& T, int i, int dep) {
  T.depth[i] = dep;
  if (T.left[i] < 0) { T.height[i] = 0; T.dims[i] = 1; }
  else {
    const int hl = finish_tree(T, T.left[i], dep + 1), hr = finish_tree(T, T.right[i], dep + 1);
    T.height[i] = 1 + (hl > hr ? hl : hr);
    T.dims[i] = T.dims[T.left[i]] + T.dims[T.right[i]];
  }
  if (T.height[i] > T.H) T.H = T.height[i];
  return T.height[i];
}

static int tree_from_arrays(int n, const int* parent, const int* left, const int* right, Tree& T) {
  if (n < 3 || n > 31 || !parent || !left || !right || parent[0] != -1) return TP_EINVAL;
  memset(&T, 0, sizeof(T));
  T.n = n;
  int seen[32] = {0};
  for (int i = 0; i < n; ++i) {
    const bool leaf = left[i] < 0;
    if (leaf != (right[i] < 0)) return TP_EINVAL;
    if (i > 0 && (parent[i] < 0 || parent[i] >= n)) return TP_EINVAL;
    T.parent[i] = parent[i]; T.left[i] = left[i]; T.right[i] = right[i];
    if (!leaf) {
      if (left[i] >= n || right[i] >= n || left[i] == right[i] || parent[left[i]] != i || parent[right[i]] != i)
        return TP_EINVAL;
      if (seen[left[i]]++ || seen[right[i]]++) return TP_EINVAL;
      T.slot[i] = T.nint++;
    } else {
      T.slot[i] = T.nleaf++;
    }
  }
  for (int i = 1; i < n; ++i) if (seen[i] != 1) return TP_EINVAL;   // every non-root node has one parent
  if (T.nleaf != T.nint + 1) return TP_EINVAL;
  finish_tree(T, 0, 0);
  return TP_OK;
}

static void plan_ht_tree(const Tree& T, int Q, int k, int nb, int r_max, HtPlan& P) {
  P.T = T;
  const int d = T.nleaf;
  P.d = d; P.Q = Q; P.k = k; P.nb = nb;
  P.ro = r_max < k ? r_max : k;
  int maxw = 1;
  for (int h = 1; h <= P.T.H; ++h) {
    int c = 0;
    for (int t = 0; t < P.T.n; ++t) if (P.T.left[t] >= 0 && P.T.height[t] == h) ++c;
    maxw = c > maxw ? c : maxw;
  }
  for (int dp = 0; dp <= P.T.H; ++dp) {
    int c = 0;
    for (int t = 0; t < P.T.n; ++t) if (P.T.left[t] >= 0 && P.T.depth[t] == dp) ++c;
    maxw = c > maxw ? c : maxw;
  }
  P.maxw = maxw;
  const size_t k3 = (size_t)k * k * k;
  size_t big = (size_t)nb * maxw * k3;
  const size_t proj = (size_t)nb * P.T.nint * (size_t)k * k * P.ro;
  const size_t nn = P.T.n, kk = (size_t)k * k;
  P.big = big > proj ? big : proj;
  if (P.big < 2 * (size_t)nb * nn * kk) P.big = 2 * (size_t)nb * nn * kk;   // F and Fi of every node (big3)
  P.off_n = (size_t)nb * (P.T.nleaf + P.T.nint) * 3 * 8 * 8;   // generous offset-table space
  P.total = align_up(8 * nb * nn * kk) * 5 + align_up(8 * nb * nn * k) * 2 + align_up(8 * nb * nn * (size_t)k * P.ro) * 2 +
            2 * align_up(4 * nb * nn) + align_up(8 * nb * nn) + 3 * align_up(8 * P.big) + align_up(8 * P.off_n) + 256 +
            align_up(8 * HT_PART);
}

static void plan_ht(int d, int Q, int k, int nb, int r_max, HtPlan& P) {
  Tree T;
  memset(&T, 0, sizeof(T));
  build_tree(T, 0, d, -1, 0);
  plan_ht_tree(T, Q, k, nb, r_max, P);
}

}  // namespace tp

using namespace tp;

static int g_split_waves = 4;   // debug hook: split-K until tiles x splits >= waves x 148 CTAs
static int g_jac_sweeps = 30;
static double g_jac_tol = 1e-16;
static int* g_jac_count = nullptr;
static int g_chol = 1;   // debug hook: 0 = eigh of every frame Gram (reference path)
static int g_form_gemm = 1;   // debug hook: 0 = node Grams / kept bases by the one-CTA form_g / form_st kernels
static int g_jac_db = 2;  // debug hook: 0 = three-barrier rows/columns, 1 = double-buffered blocks, 2 = upper-triangle blocks (default)
static int g_eig_tridiag = 1;   // debug hook: node-Gram eigensolver 1 = tridiagonal (default), 0 = Jacobi (g_jac_db)

extern "C" {

// debug hook: Jacobi sweep cap, rotation threshold, optional device counter of sweeps done
void tp_debug_set_jacobi(int max_sweeps, double tol, int* count) {
  g_jac_sweeps = max_sweeps; g_jac_tol = tol; g_jac_count = count;
}
// debug hook: batched-GEMM kernel variant of the hSVD chain (tp_gemm.cuh g_bgemm_variant)
void tp_debug_set_bgemm_variant(int v) { g_bgemm_variant = v; }
void tp_debug_set_ht_split_waves(int w) { g_split_waves = w; }
void tp_debug_set_bgemm_klayout(int on) { g_bgemm_klayout = on; }
// debug hook: frame-Gram factor by Cholesky (1, default) or eigh (0)
void tp_debug_set_ht_chol(int on) { g_chol = on; }
void tp_debug_set_ht_form_gemm(int on) { g_form_gemm = on; }
// debug hook: Jacobi kernel (0 = three-barrier rounds, 1 = double-buffered blocks, 2 = upper-triangle blocks, default)
void tp_debug_set_jacobi_impl(int db) { g_jac_db = db; }
// debug hook: node-Gram eigensolver (1 = Householder tridiagonal + bisection + inverse iteration, 0 = Jacobi)
void tp_debug_set_eig_tridiag(int on) { g_eig_tridiag = on; }

size_t tp_ht_truncate_ws_bytes(int d, int Q, int k, int nb) {
  if (d < 2 || d > 16 || Q < 1 || k < 1 || k > 64 || nb < 1) return 0;
  HtPlan P;
  plan_ht(d, Q, k, nb, k, P);
  return P.total;
}

static int ht_truncate_impl(const Tree& TT, int Q, int k, int nb, const double* frames, const double* transfers,
                            int r_max, double eps, double* out_frames, double* out_transfers, int* out_ranks,
                            double* est, double* norms, void* ws, size_t ws_bytes, void* stream);

int tp_ht_truncate_f64(int d, int Q, int k, int nb, const double* frames, const double* transfers,
                       int r_max, double eps, double* out_frames, double* out_transfers,
                       int* out_ranks, double* est, double* norms,
                       void* ws, size_t ws_bytes, void* stream) {
  if (d < 2 || d > 16) return TP_EINVAL;
  Tree T;
  memset(&T, 0, sizeof(T));
  build_tree(T, 0, d, -1, 0);
  return ht_truncate_impl(T, Q, k, nb, frames, transfers, r_max, eps, out_frames, out_transfers, out_ranks, est,
                          norms, ws, ws_bytes, stream);
}

size_t tp_ht_truncate_tree_ws_bytes(int n_nodes, const int* parent, const int* left, const int* right, int Q, int k,
                                    int nb) {
  Tree T;
  if (tree_from_arrays(n_nodes, parent, left, right, T) != TP_OK || Q < 1 || k < 1 || k > 64 || nb < 1) return 0;
  HtPlan P;
  plan_ht_tree(T, Q, k, nb, k, P);
  return P.total;
}

int tp_ht_truncate_tree_f64(int n_nodes, const int* parent, const int* left, const int* right, int Q, int k, int nb,
                            const double* frames, const double* transfers, int r_max, double eps,
                            double* out_frames, double* out_transfers, int* out_ranks, double* est, double* norms,
                            void* ws, size_t ws_bytes, void* stream) {
  Tree T;
  const int st = tree_from_arrays(n_nodes, parent, left, right, T);
  if (st != TP_OK) return st;
  return ht_truncate_impl(T, Q, k, nb, frames, transfers, r_max, eps, out_frames, out_transfers, out_ranks, est,
                          norms, ws, ws_bytes, stream);
}

}  // extern "C"

static int ht_truncate_impl(const Tree& TT, int Q, int k, int nb, const double* frames, const double* transfers,
                            int r_max, double eps, double* out_frames, double* out_transfers, int* out_ranks,
                            double* est, double* norms, void* ws, size_t ws_bytes, void* stream) {
  const int d = TT.nleaf;
  if (d < 2 || d > 16 || Q < 1 || k < 1 || nb < 1 || r_max < 1 || !(eps >= 0.0)) return TP_EINVAL;
  if (!frames || !transfers || !out_frames || !out_transfers || !out_ranks || !est || !norms) return TP_EINVAL;
  if (k > 64) return TP_EUNSUPPORTED;
  HtPlan P;
  plan_ht_tree(TT, Q, k, nb, r_max, P);
  HtPlan P0;
  plan_ht_tree(TT, Q, k, nb, k, P0);
  if (!ws || ws_bytes < P0.total) return TP_EWORKSPACE;
  const Tree& T = P.T;
  const int nn = T.n, ro = P.ro;
  const long long kk = (long long)k * k, k3 = kk * k;
  cudaStream_t st = (cudaStream_t)stream;
  Carver cv(ws, ws_bytes);
  double* Mf = cv.take<double>((size_t)nb * nn * kk);
  double* Gh = cv.take<double>((size_t)nb * nn * kk);
  double* Vm = cv.take<double>((size_t)nb * nn * kk);
  double* Wg = cv.take<double>((size_t)nb * nn * kk);
  double* Gt = cv.take<double>((size_t)nb * nn * kk);
  double* lam = cv.take<double>((size_t)nb * nn * k);
  double* sig = cv.take<double>((size_t)nb * nn * k);
  double* S = cv.take<double>((size_t)nb * nn * k * ro);
  double* Tm = cv.take<double>((size_t)nb * nn * ro * k);
  int* keep = cv.take<int>((size_t)nb * nn);
  int* cholok = cv.take<int>((size_t)nb * nn);
  double* disc = cv.take<double>((size_t)nb * nn);
  double* big1 = cv.take<double>(P0.big);
  double* big2 = cv.take<double>(P0.big);
  double* big3 = cv.take<double>(P0.big);
  long long* doffs = cv.take<long long>(P0.off_n);
  double* kpart = cv.take<double>(HT_PART);
  double* one = reinterpret_cast<double*>(cv.take<double>(1));
  if (!cv.ok()) return TP_EWORKSPACE;

  // all offset tables are built on the host and uploaded once
  std::vector<long long> hoffs;
  auto table = [&](const std::vector<long long>& v) {
    const size_t at = hoffs.size();
    hoffs.insert(hoffs.end(), v.begin(), v.end());
    return at;
  };
  auto MF = [&](int b, int t) { return ((long long)b * nn + t) * kk; };
  auto BT = [&](int b, int t) { return ((long long)b * T.nint + T.slot[t]) * k3; };
  auto UF = [&](int b, int t) { return ((long long)b * T.nleaf + T.slot[t]) * (long long)Q * k; };

  struct Call { BGemm g; size_t tab; int use_tab; };
  std::vector<Call> calls;
  std::vector<int> kinds;   // 0 = gemm, 1 = transpose(kt, tab, nb1), 2 = marker for non-gemm stage
  struct Tr { int kt; size_t tab; int n; };
  std::vector<Tr> trs;
  std::vector<int> order;   // sequence of (kind) entries referencing calls / trs / stages
  // stage ids: -1 eigh(M), -2 set_root_env, -3 form_g, -4 eigh(G), -5 keep, -6 form_st, -7 finish
  auto add_gemm = [&](BGemm g, const std::vector<long long>& offs) {
    Call c{g, 0, 0};
    if (!offs.empty()) { c.tab = table(offs); c.use_tab = 1; c.g.nb1 = (int)(offs.size() / 3); }
    const int ks = bgemm_pick_split(c.g, 148, 8, g_split_waves);
    if (ks > 1 && (size_t)c.g.M * c.g.N * c.g.nb1 * c.g.nb2 * ks <= HT_PART) { c.g.ksplit = ks; c.g.part = kpart; }
    calls.push_back(c);
    order.push_back((int)calls.size() - 1);
  };
  auto add_stage = [&](int id) { order.push_back(id); };

  // ---- 1. frame Grams, leaves -> root
  {
    std::vector<long long> o;
    for (int b = 0; b < nb; ++b)
      for (int t = 0; t < nn; ++t)
        if (T.left[t] < 0) { o.push_back(UF(b, t)); o.push_back(UF(b, t)); o.push_back(MF(b, t)); }
    add_gemm(bgemm_desc(k, k, Q, frames, 1, k, frames, k, 1, Mf, k, 1), o);
  }
  for (int h = 1; h <= T.H; ++h) {
    std::vector<int> W;
    for (int t = 0; t < nn; ++t) if (T.left[t] >= 0 && T.height[t] == h) W.push_back(t);
    if (W.empty()) continue;
    for (int kt : {k, 1}) {
      std::vector<int> Wk;
      for (int t : W) if ((t == 0 ? 1 : k) == kt) Wk.push_back(t);
      if (Wk.empty()) continue;
      std::vector<long long> o1, o2, o3;
      int zz = 0;
      for (int b = 0; b < nb; ++b)
        for (int t : Wk) {
          const long long zb = (long long)zz++ * k3;
          o1.insert(o1.end(), {MF(b, T.left[t]), BT(b, t), zb});                 // T1 = M_l B
          o2.insert(o2.end(), {MF(b, T.right[t]), zb, zb});                      // T2[c] = M_r T1[c]
          o3.insert(o3.end(), {BT(b, t), zb, MF(b, t)});                         // M_t = B^T T2
        }
      BGemm g1 = bgemm_desc(k, k * kt, k, Mf, k, 1, transfers, (long long)k * kt, 1, big1, (long long)k * kt, 1);
      add_gemm(g1, o1);
      BGemm g2 = bgemm_desc(k, kt, k, Mf, k, 1, big1, kt, 1, big2, kt, 1);
      g2.nb2 = k; g2.sA2 = 0; g2.sB2 = (long long)k * kt; g2.sC2 = (long long)k * kt;
      add_gemm(g2, o2);
      BGemm g3 = bgemm_desc(kt, kt, k * k, transfers, 1, kt, big2, kt, 1, Mf, kt, 1);
      add_gemm(g3, o3);
    }
  }
  add_stage(-1);   // eigh of frame Grams (non-root)
  add_stage(-2);   // Gh_root = 1
  // ---- 2. environment Grams, root -> leaves
  for (int dp = 0; dp < T.H; ++dp) {
    for (int kt : {k, 1}) {
      std::vector<int> Wk;
      for (int t = 0; t < nn; ++t)
        if (T.left[t] >= 0 && T.depth[t] == dp && (t == 0 ? 1 : k) == kt) Wk.push_back(t);
      if (Wk.empty()) continue;
      std::vector<long long> oX, oY, oGl, oZ, oTr, oGr;
      int zz = 0;
      for (int b = 0; b < nb; ++b)
        for (int t : Wk) {
          const long long zb = (long long)zz++ * k3;
          oX.insert(oX.end(), {BT(b, t), MF(b, t), zb});                          // X = B Gh_t
          oY.insert(oY.end(), {MF(b, T.right[t]), zb, zb});                       // Y[a] = M_r X[a]
          oGl.insert(oGl.end(), {zb, BT(b, t), MF(b, T.left[t])});                // Gh_l = Y B^T
          oZ.insert(oZ.end(), {MF(b, T.left[t]), zb, zb});                        // Z'[b'] = M_l X[:, b', :]
          oTr.insert(oTr.end(), {BT(b, t), 0, 0});
          oGr.insert(oGr.end(), {zb, (kt == 1 || kt % 16 == 0) ? BT(b, t) : zb, MF(b, T.right[t])});   // Gh_r
        }
      const long long kkt = (long long)k * kt;
      BGemm gX = bgemm_desc(k * k, kt, kt, transfers, kt, 1, Gh, kt, 1, big1, kt, 1);
      add_gemm(gX, oX);
      BGemm gY = bgemm_desc(k, kt, k, Mf, k, 1, big1, kt, 1, big2, kt, 1);
      gY.nb2 = k; gY.sA2 = 0; gY.sB2 = kkt; gY.sC2 = kkt;
      add_gemm(gY, oY);
      BGemm gGl = bgemm_desc(k, k, k * kt, big2, kkt, 1, transfers, 1, kkt, Gh, k, 1);
      add_gemm(gGl, oGl);
      BGemm gZ = bgemm_desc(k, kt, k, Mf, k, 1, big1, kkt, 1, big2, kt, 1);
      gZ.nb2 = k; gZ.sA2 = 0; gZ.sB2 = kt; gZ.sC2 = kkt;
      add_gemm(gZ, oZ);
      // Gh_r[b][b'] = sum_{a,j} Z'[b][a][j] B[a][b'][j]: B read in place, K = (a, j) by the
      // two-level K addressing (no transposed copy of B)
      // (k-tiles must not straddle two runs of kt: otherwise the transposed copy Bp[b][a][j])
      BGemm gGr;
      if (kt == 1) {
        gGr = bgemm_desc(k, k, k, big2, kkt, 1, transfers, k, 1, Gh, k, 1);
      } else if (kt % 16 == 0) {
        gGr = bgemm_desc(k, k, k * kt, big2, kkt, 1, transfers, 1, kt, Gh, k, 1);
        gGr.kinB = kt;
        gGr.sBk1 = (long long)k * kt;
      } else {
        trs.push_back({kt, table(oTr), (int)(oTr.size() / 3)});
        order.push_back(-100 - (int)(trs.size() - 1));
        gGr = bgemm_desc(k, k, k * kt, big2, kkt, 1, big3, 1, kkt, Gh, k, 1);
      }
      add_gemm(gGr, oGr);
    }
  }
  // node Grams G_t = F^T Gh F, then S_t = Fi^T W_keep, T_t = W_keep^T F^T as batched GEMMs over
  // every non-root node (F, Fi from frame_factor_kernel in the big3 scratch; P in big1)
  const long long nodes_kk = (long long)nb * nn * kk;
  std::vector<long long> oP, oG, oS, oT;
  for (int b = 0; b < nb; ++b)
    for (int t = 1; t < nn; ++t) {
      const long long nd = ((long long)b * nn + t) * kk;
      oP.insert(oP.end(), {nd, nd, nd});                                                   // P = F^T Gh
      oG.insert(oG.end(), {nd, nd, nd});                                                   // G = P F
      oS.insert(oS.end(), {nd, nd, ((long long)b * nn + t) * k * ro});                     // S = Fi^T W
      oT.insert(oT.end(), {nd, nd, ((long long)b * nn + t) * ro * k});                     // T = W^T F^T
    }
  if (g_form_gemm) {
    add_stage(-8);   // F, Fi
    add_gemm(bgemm_desc(k, k, k, big3, 1, k, Gh, k, 1, big1, k, 1), oP);
    add_gemm(bgemm_desc(k, k, k, big1, k, 1, big3, k, 1, Gt, k, 1), oG);
  } else {
    add_stage(-3);   // G_t = L^1/2 V^T Gh V L^1/2
  }
  add_stage(-4);   // eigh(G_t)
  add_stage(-5);   // keep rule
  if (g_form_gemm) {
    add_gemm(bgemm_desc(k, ro, k, big3 + nodes_kk, 1, k, Wg, k, 1, S, ro, 1), oS);
    add_gemm(bgemm_desc(ro, k, k, Wg, 1, k, big3, 1, k, Tm, k, 1), oT);
  } else {
    add_stage(-6);   // S_t, T_t
  }
  add_stage(-7);   // est, norms, ranks
  // ---- 4. projection
  {
    std::vector<long long> o;
    for (int b = 0; b < nb; ++b)
      for (int t = 0; t < nn; ++t)
        if (T.left[t] < 0)
          o.insert(o.end(), {UF(b, t), ((long long)b * nn + t) * k * ro, ((long long)b * T.nleaf + T.slot[t]) * Q * ro});
    add_gemm(bgemm_desc(Q, ro, k, frames, k, 1, S, ro, 1, out_frames, ro, 1), o);
  }
  for (int kt : {k, 1}) {
    const int rt = (kt == 1) ? 1 : ro;
    std::vector<long long> o1, o2, o3;
    int zz = 0;
    for (int b = 0; b < nb; ++b)
      for (int t = 0; t < nn; ++t) {
        if (T.left[t] < 0 || (t == 0 ? 1 : k) != kt) continue;
        const long long zb = (long long)zz++ * k * k * ro;
        const long long sOff = ((long long)b * nn + t) * k * ro;
        o1.insert(o1.end(), {BT(b, t), kt == 1 ? 0 : sOff, zb});                                  // X1 = B S_t
        o2.insert(o2.end(), {((long long)b * nn + T.left[t]) * ro * k, zb, zb});                 // X2 = T_l X1
        o3.insert(o3.end(), {((long long)b * nn + T.right[t]) * ro * k, zb,
                             ((long long)b * T.nint + T.slot[t]) * (long long)ro * ro * ro});    // B'[c] = T_r X2[c]
      }
    if (o1.empty()) continue;
    BGemm g1 = (kt == 1) ? bgemm_desc(k * k, 1, 1, transfers, 1, 1, one, 0, 0, big1, 1, 1)
                         : bgemm_desc(k * k, ro, k, transfers, k, 1, S, ro, 1, big1, ro, 1);
    add_gemm(g1, o1);
    BGemm g2 = bgemm_desc(ro, k * rt, k, Tm, k, 1, big1, (long long)k * rt, 1, big2, (long long)k * rt, 1);
    add_gemm(g2, o2);
    BGemm g3 = bgemm_desc(ro, rt, k, Tm, k, 1, big2, rt, 1, out_transfers, rt, 1);
    g3.nb2 = ro; g3.sA2 = 0; g3.sB2 = (long long)k * rt; g3.sC2 = (long long)ro * rt;
    add_gemm(g3, o3);
  }

  if (hoffs.size() > P0.off_n) return TP_EWORKSPACE;
  // offset tables and the structural rank bounds: uploaded once per shape and cached on
  // the device (no pageable copies: the call is stream-ordered and graph-capturable)
  // hb: rank of the node's frame (subtree matricization); cb: rank bound of the complement;
  // the node Gram's rank is <= min(hb, cb) -- eigenvalues past it are exactly zero in the
  // reference's arithmetic (dropped by its keep rule) and rounding noise here
  std::vector<int> hb(nn, k), cb(nn, k), bnd(2 * nn, k);
  for (int t = nn - 1; t >= 0; --t)
    hb[t] = T.left[t] < 0 ? (Q < k ? Q : k)
                          : ((long long)hb[T.left[t]] * hb[T.right[t]] < k ? hb[T.left[t]] * hb[T.right[t]] : k);
  for (int t = 0; t < nn; ++t) {
    if (T.left[t] < 0) continue;
    const int l = T.left[t], r = T.right[t];
    const long long cl = (t == 0) ? hb[r] : (long long)cb[t] * hb[r], cr = (t == 0) ? hb[l] : (long long)cb[t] * hb[l];
    cb[l] = cl < k ? (int)cl : k;
    cb[r] = cr < k ? (int)cr : k;
  }
  for (int t = 0; t < nn; ++t) {
    bnd[t] = hb[t];                                    // frame-Gram pseudo-inverse (form_g, form_st)
    bnd[nn + t] = hb[t] < cb[t] ? hb[t] : cb[t];       // node-Gram keep bound (keep_rule)
  }
  bnd[0] = bnd[nn] = 1;
  const int* bound = device_table(bnd);
  const long long* dtab = device_table(hoffs);
  const double* one_c = device_table(std::vector<double>{1.0});
  if (!bound || !dtab || !one_c) return TP_ECUDA;
  (void)doffs;
  cudaError_t e = cudaMemcpyAsync(one, one_c, sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_status(e);
  e = cudaMemsetAsync(Gh, 0, sizeof(double) * (size_t)nb * nn * kk, st);
  if (e != cudaSuccess) return cuda_status(e);

  const int kp = k + (k & 1);
  const size_t jsm = g_jac_db == 1 ? sizeof(double) * (size_t)3 * kp * (kp + 1)
                   : g_jac_db == 2 ? sizeof(double) * ((size_t)kp * (kp + 1) / 2 + (size_t)kp * (kp + 1) + 2 * 32 * 3) +
                                         sizeof(int) * (2 * 32 * 2 + 2) +
                                         sizeof(unsigned short) * 33 * 32 / 2 + 16
                                   : sizeof(double) * ((size_t)2 * kp * (kp + 1) + 2 * kp + JAC_NT) + sizeof(int) * kp;
  auto jac = g_jac_db == 1 ? jacobi_db_kernel : (g_jac_db == 2 ? jacobi_sym_kernel : jacobi_eigh_kernel);
  cudaFuncSetAttribute(jac, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jsm);
  const size_t fsm = sizeof(double) * 3 * (size_t)k * (k + 1);
  cudaFuncSetAttribute(form_g_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  const size_t ssm = sizeof(double) * ((size_t)k + 2 * (size_t)k * ro + (size_t)k * (k + 1) + (size_t)k);
  cudaFuncSetAttribute(form_st_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
  const size_t ffsm = sizeof(double) * (2 * (size_t)k * (k + 1) + (size_t)k);
  cudaFuncSetAttribute(frame_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ffsm);
  const size_t csm = sizeof(double) * ((size_t)k * (k + (((4 - k % 16) + 16) % 16)) + 2);
  cudaFuncSetAttribute(chol_frame_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  const int nonroot = nb * (nn - 1);
  for (int id : order) {
    if (id >= 0) {
      BGemm g = calls[id].g;
      if (calls[id].use_tab) g.offs = dtab + calls[id].tab;
      e = bgemm_launch(g, st);
    } else if (id <= -100) {
      const Tr& tr = trs[-100 - id];
      dim3 grid(64, tr.n);
      transpose12_kernel<<<grid, 256, 0, st>>>(k, tr.kt, dtab + tr.tab, transfers, big3, k3);
      e = cudaGetLastError();
    } else if (id == -1) {
      if (g_chol) {
        chol_frame_kernel<<<nonroot, 256, csm, st>>>(k, nn, Mf, Vm, cholok);
      } else {
        e = cudaMemsetAsync(cholok, 0, sizeof(int) * (size_t)nb * nn, st);
        if (e != cudaSuccess) return cuda_status(e);
      }
      jac<<<nonroot, JAC_NT, jsm, st>>>(k, nn, 1, nn - 1, Mf, Vm, lam, g_jac_sweeps, g_jac_tol, g_jac_count,
                                                        cholok);
      e = cudaGetLastError();
    } else if (id == -2) {
      set_root_env<<<(nb + 127) / 128, 128, 0, st>>>(k, nn, nb, Gh);
      e = cudaGetLastError();
    } else if (id == -3) {
      form_g_kernel<<<nonroot, 256, fsm, st>>>(k, nn, Vm, lam, Gh, Gt, cholok, bound);
      e = cudaGetLastError();
    } else if (id == -4) {
      if (g_eig_tridiag) {   // eigenvalues + the ro kept eigenvectors: tridiagonalisation (tp_eigh.cu)
        e = launch_tridiag_eigh(nonroot, k, nn, 1, nn - 1, Gt, Wg, sig, P.ro, nullptr, st);
      } else {
        jac<<<nonroot, JAC_NT, jsm, st>>>(k, nn, 1, nn - 1, Gt, Wg, sig, g_jac_sweeps, g_jac_tol, g_jac_count,
                                                          nullptr);
        e = cudaGetLastError();
      }
    } else if (id == -5) {
      keep_rule_kernel<<<(nonroot + 127) / 128, 128, 0, st>>>(k, nn, nb, d, eps, r_max, sig, Mf, keep, disc, bound,
                                                               g_form_gemm ? Wg : nullptr, ro);
      e = cudaGetLastError();
    } else if (id == -8) {
      frame_factor_kernel<<<nonroot, 256, ffsm, st>>>(k, nn, Vm, lam, cholok, bound, big3, big3 + nodes_kk);
      e = cudaGetLastError();
    } else if (id == -6) {
      form_st_kernel<<<nonroot, 256, ssm, st>>>(k, ro, nn, Vm, lam, Wg, keep, Mf, S, Tm, cholok, bound);
      e = cudaGetLastError();
    } else if (id == -7) {
      finish_kernel<<<(nb + 127) / 128, 128, 0, st>>>(k, nn, nb, Mf, keep, disc, est, norms, out_ranks);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) return cuda_status(e);
  }
  return TP_OK;
}
