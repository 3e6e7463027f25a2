// Batched, arbitrarily-strided fp64 GEMM on the DMMA tensor pipe (sm_100a):
//   C_z(m, n) = alpha * sum_k A_z(m, k) B_z(k, n) + beta * C_z(m, n)
// Element (m, k) of A_z sits at A + offA(z) + m*sAm + k*sAk (same for B, C), so
// transposes, tensor-mode contractions and Kronecker-style batched products are
// all strided views -- no data is ever transposed in memory.
// Batch z = (z1, z2): z1 indexes an optional device table of base offsets
// (3 per entry: A, B, C) or uniform strides; z2 is an inner uniform batch.
#pragma once
#include "tp_common.cuh"

namespace tp {

constexpr int GB_TM = 64, GB_TN = 64, GB_TK = 16, GB_LD = 68;   // 68 == 4 (mod 16): conflict-free fragments

struct BGemm {
  int M, N, K, nb1, nb2;
  long long sAm, sAk, sBk, sBn, sCm, sCn;
  long long sA1, sB1, sC1;   // outer batch strides (used when offs == nullptr)
  long long sA2, sB2, sC2;   // inner batch strides
  const long long* offs;     // [nb1][3] base offsets or nullptr
  const double* A;
  const double* B;
  double* C;
  double alpha, beta;
  int ksplit;                // split-K factor (>1: partial tiles to `part`, then bgemm_reduce)
  double* part;              // [nb1*nb2][ksplit][M][N] partials when ksplit > 1
  const int* skip;           // optional device flag: nonzero -> the launch is a no-op (stream-ordered early exit)
  // two-level K addressing of a K-contiguous B (pipelined kernel only): k -> (k / kinB) * sBk1 + k % kinB,
  // e.g. the (a, j) pairs of a transfer tensor B[a][b][j] read for fixed b without a transpose
  int kinB;                  // 0: plain k * sBk
  long long sBk1;
};

// 8-byte global -> shared async copy (LDGSTS); src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(valid ? src : nullptr), "r"(valid ? 8 : 0)
               : "memory");
}

static __global__ void __launch_bounds__(128) bgemm_kernel(const __grid_constant__ BGemm g) {
  if (g.skip && *g.skip) return;
  // two-stage cp.async pipeline: K tile t+1 streams into the other buffer while
  // tile t is multiplied on the DMMA pipe
  __shared__ double As[2][GB_TK][GB_LD];
  __shared__ double Bs[2][GB_TK][GB_LD];
  const int ks = g.ksplit > 1 ? g.ksplit : 1;
  const int zz = blockIdx.z / ks, sidx = blockIdx.z - zz * ks;
  const int z1 = zz / g.nb2, z2 = zz % g.nb2;
  long long oA, oB, oC;
  if (g.offs) {
    oA = g.offs[3 * z1]; oB = g.offs[3 * z1 + 1]; oC = g.offs[3 * z1 + 2];
  } else {
    oA = z1 * g.sA1; oB = z1 * g.sB1; oC = z1 * g.sC1;
  }
  const double* A = g.A + oA + z2 * g.sA2;
  const double* B = g.B + oB + z2 * g.sB2;
  double* C = g.C + oC + z2 * g.sC2;
  const int m0 = blockIdx.y * GB_TM, n0 = blockIdx.x * GB_TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const bool a_m_fast = g.sAm == 1, b_n_fast = g.sBn == 1;
  // split-K range of this CTA (whole GB_TK tiles)
  const int ktiles = (g.K + GB_TK - 1) / GB_TK, kt0 = (int)((long long)ktiles * sidx / ks),
            kt1 = (int)((long long)ktiles * (sidx + 1) / ks);
  auto issue = [&](int kt, int buf) {
    const int k0 = kt * GB_TK;
#pragma unroll 2
    for (int e = tid; e < GB_TK * GB_TM; e += 128) {
      int kk, mm;
      if (a_m_fast) { kk = e / GB_TM; mm = e % GB_TM; } else { mm = e / GB_TK; kk = e % GB_TK; }
      const int m = m0 + mm, k = k0 + kk;
      const bool v = m < g.M && k < g.K;
      cp_async8(&As[buf][kk][mm], A + (v ? m * g.sAm + k * g.sAk : 0), v);
    }
#pragma unroll 2
    for (int e = tid; e < GB_TK * GB_TN; e += 128) {
      int kk, nn;
      if (b_n_fast) { kk = e / GB_TN; nn = e % GB_TN; } else { nn = e / GB_TK; kk = e % GB_TK; }
      const int n = n0 + nn, k = k0 + kk;
      const bool v = n < g.N && k < g.K;
      cp_async8(&Bs[buf][kk][nn], B + (v ? k * g.sBk + n * g.sBn : 0), v);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if (kt0 < kt1) issue(kt0, 0);
  for (int kt = kt0; kt < kt1; ++kt) {
    const int buf = (kt - kt0) & 1;
    if (kt + 1 < kt1) {
      issue(kt + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int ksub = 0; ksub < GB_TK; ksub += 4) {
      const int kr = ksub + (lane & 3), cc = lane >> 2;
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = As[buf][kr][wm + 8 * i + cc];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = Bs[buf][kr][wn + 8 * j + cc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
    __syncthreads();   // buffer `buf` is refilled by the next iteration's issue
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + 8 * i + (lane >> 2), n = n0 + wn + 8 * j + 2 * (lane & 3) + h;
        if (m < g.M && n < g.N) {
          if (ks > 1) {
            g.part[(((size_t)zz * ks + sidx) * g.M + m) * g.N + n] = acc[i][j][h];
          } else {
            double* c = C + m * g.sCm + n * g.sCn;
            const double v = g.alpha * acc[i][j][h];
            *c = (g.beta == 0.0) ? v : fma(g.beta, *c, v);
          }
        }
      }
}

// 16-byte global -> shared async copy (LDGSTS.128)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// Same tiling and fragment schedule as bgemm_kernel (64 x 64 tile, 4 warps of
// 32 x 32, m8n8k4 DMMA), with a STAGES-deep cp.async ring of TK-deep K tiles in
// dynamic shared memory and 16-byte copies along a contiguous, 16-byte aligned
// M (A) / N (B) dimension.
// AK / BK: operand stored K-contiguous in global memory (sAk == 1 / sBk == 1 with the
// other stride != 1): the tile is kept [m][k] in shared memory (row stride TK + 4,
// conflict-free fragments) and filled with 16-byte copies along K.
template <int STAGES, int TK, bool AK = false, bool BK = false>
static __global__ void __launch_bounds__(128) bgemm_pipe_kernel(const __grid_constant__ BGemm g) {
  if (g.skip && *g.skip) return;
  extern __shared__ double gsm[];
  constexpr int LDK = TK + 4;
  constexpr int SA = AK ? GB_TM * LDK : TK * GB_LD, SB = BK ? GB_TN * LDK : TK * GB_LD;   // per stage
  double* As = gsm;                                  // [STAGES][SA]
  double* Bs = gsm + (size_t)STAGES * SA;            // [STAGES][SB]
  const int ks = g.ksplit > 1 ? g.ksplit : 1;
  const int zz = blockIdx.z / ks, sidx = blockIdx.z - zz * ks;
  const int z1 = zz / g.nb2, z2 = zz % g.nb2;
  long long oA, oB, oC;
  if (g.offs) {
    oA = g.offs[3 * z1]; oB = g.offs[3 * z1 + 1]; oC = g.offs[3 * z1 + 2];
  } else {
    oA = z1 * g.sA1; oB = z1 * g.sB1; oC = z1 * g.sC1;
  }
  const double* A = g.A + oA + z2 * g.sA2;
  const double* B = g.B + oB + z2 * g.sB2;
  double* C = g.C + oC + z2 * g.sC2;
  const int m0 = blockIdx.y * GB_TM, n0 = blockIdx.x * GB_TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const bool a_m_fast = g.sAm == 1, b_n_fast = g.sBn == 1;
  const bool a_vec = a_m_fast && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (g.sAk % 2 == 0);
  const bool b_vec = b_n_fast && ((reinterpret_cast<uintptr_t>(B) & 15) == 0) && (g.sBk % 2 == 0);
  const int ktiles = (g.K + TK - 1) / TK, kt0 = (int)((long long)ktiles * sidx / ks),
            kt1 = (int)((long long)ktiles * (sidx + 1) / ks);
  auto load_tile = [&](const double* X, long long sXi, long long sXk, int I, int i0, bool fast, bool vec, double* dst,
                       int k0) {
    if (vec) {
#pragma unroll 2
      for (int e = tid; e < TK * GB_TM / 2; e += 128) {
        const int kk = e / (GB_TM / 2), ii = 2 * (e % (GB_TM / 2));
        const int i = i0 + ii, k = k0 + kk;
        double* d = dst + kk * GB_LD + ii;
        if (k < g.K && i + 1 < I) {
          cp_async16(d, X + i + k * sXk);
        } else {
          cp_async8(d, X + ((i < I && k < g.K) ? i + k * sXk : 0), i < I && k < g.K);
          cp_async8(d + 1, X + ((i + 1 < I && k < g.K) ? i + 1 + k * sXk : 0), i + 1 < I && k < g.K);
        }
      }
    } else {
#pragma unroll 2
      for (int e = tid; e < TK * GB_TM; e += 128) {
        int kk, ii;
        if (fast) { kk = e / GB_TM; ii = e % GB_TM; } else { ii = e / TK; kk = e % TK; }
        const int i = i0 + ii, k = k0 + kk;
        const bool v = i < I && k < g.K;
        cp_async8(dst + kk * GB_LD + ii, X + (v ? i * sXi + k * sXk : 0), v);
      }
    }
  };
  // K-contiguous operand -> [i][k] tile (row stride LDK), 16-byte copies of k pairs
  auto load_tile_k = [&](const double* X, long long sXi, int I, int i0, bool vec, double* dst, int k0, int kin,
                         long long sk1) {
    // (kin > 0: the k-tile lies inside one run of kin contiguous k, kin a multiple of TK)
    const long long kb = kin > 0 ? (long long)(k0 / kin) * sk1 + (k0 % kin) - k0 : 0;
#pragma unroll 2
    for (int e = tid; e < GB_TM * TK / 2; e += 128) {
      const int ii = e / (TK / 2), kk = 2 * (e % (TK / 2));
      const int i = i0 + ii, k = k0 + kk;
      double* d = dst + ii * LDK + kk;
      if (vec && i < I && k + 1 < g.K) {
        cp_async16(d, X + i * sXi + k + kb);
      } else {
        cp_async8(d, X + ((i < I && k < g.K) ? i * sXi + k + kb : 0), i < I && k < g.K);
        cp_async8(d + 1, X + ((i < I && k + 1 < g.K) ? i * sXi + k + 1 + kb : 0), i < I && k + 1 < g.K);
      }
    }
  };
  const bool ak_vec = AK && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (g.sAm % 2 == 0);
  const bool bk_vec = BK && ((reinterpret_cast<uintptr_t>(B) & 15) == 0) && (g.sBn % 2 == 0);
  auto issue = [&](int kt, int buf) {
    const int k0 = kt * TK;
    if (AK) load_tile_k(A, g.sAm, g.M, m0, ak_vec, As + (size_t)buf * SA, k0, 0, 0);
    else load_tile(A, g.sAm, g.sAk, g.M, m0, a_m_fast, a_vec, As + (size_t)buf * SA, k0);
    if (BK) load_tile_k(B, g.sBn, g.N, n0, bk_vec, Bs + (size_t)buf * SB, k0, g.kinB, g.sBk1);
    else load_tile(B, g.sBn, g.sBk, g.N, n0, b_n_fast, b_vec, Bs + (size_t)buf * SB, k0);
  };
  // prologue: STAGES - 1 tiles in flight (one commit group per stage, possibly empty)
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (kt0 + st < kt1) issue(kt0 + st, st);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int kt = kt0; kt < kt1; ++kt) {
    const int it = kt - kt0, buf = it % STAGES;
    asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 2) : "memory");
    __syncthreads();   // tile `it` visible to all; the buffer refilled below is free
    if (kt + STAGES - 1 < kt1) issue(kt + STAGES - 1, (it + STAGES - 1) % STAGES);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const double* Ab = As + (size_t)buf * SA;
    const double* Bb = Bs + (size_t)buf * SB;
#pragma unroll
    for (int ksub = 0; ksub < TK; ksub += 4) {
      const int kr = ksub + (lane & 3), cc = lane >> 2;
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = AK ? Ab[(wm + 8 * i + cc) * LDK + kr] : Ab[kr * GB_LD + wm + 8 * i + cc];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = BK ? Bb[(wn + 8 * j + cc) * LDK + kr] : Bb[kr * GB_LD + wn + 8 * j + cc];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + 8 * i + (lane >> 2), n = n0 + wn + 8 * j + 2 * (lane & 3) + h;
        if (m < g.M && n < g.N) {
          if (ks > 1) {
            g.part[(((size_t)zz * ks + sidx) * g.M + m) * g.N + n] = acc[i][j][h];
          } else {
            double* c = C + m * g.sCm + n * g.sCn;
            const double v = g.alpha * acc[i][j][h];
            *c = (g.beta == 0.0) ? v : fma(g.beta, *c, v);
          }
        }
      }
}

// split-K epilogue: C_z = alpha * sum_s part[z][s] + beta * C_z (fixed order)
static __global__ void bgemm_reduce_kernel(const __grid_constant__ BGemm g) {
  if (g.skip && *g.skip) return;
  const int z = blockIdx.y, z1 = z / g.nb2, z2 = z % g.nb2;
  long long oC = g.offs ? g.offs[3 * z1 + 2] : z1 * g.sC1;
  double* C = g.C + oC + z2 * g.sC2;
  const size_t mn = (size_t)g.M * g.N;
  const double* p = g.part + (size_t)z * g.ksplit * mn;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < mn; e += (size_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < g.ksplit; ++s) acc += p[s * mn + e];
    const int m = (int)(e / g.N), n = (int)(e % g.N);
    double* c = C + m * g.sCm + n * g.sCn;
    const double v = g.alpha * acc;
    *c = (g.beta == 0.0) ? v : fma(g.beta, *c, v);
  }
}

static inline BGemm bgemm_desc(int M, int N, int K, const double* A, long long sAm, long long sAk, const double* B,
                        long long sBk, long long sBn, double* C, long long sCm, long long sCn) {
  BGemm g{};
  g.M = M; g.N = N; g.K = K; g.nb1 = 1; g.nb2 = 1;
  g.A = A; g.B = B; g.C = C;
  g.sAm = sAm; g.sAk = sAk; g.sBk = sBk; g.sBn = sBn; g.sCm = sCm; g.sCn = sCn;
  g.alpha = 1.0; g.beta = 0.0;
  g.ksplit = 1; g.part = nullptr;
  return g;
}

// split-K factor that fills the GPU (>= 2 CTAs per SM) for K-heavy batched GEMMs
static inline int bgemm_pick_split(const BGemm& g, int nsm = 148, int min_ktiles = 8, int waves = 2) {
  const long long tiles = (long long)((g.N + GB_TN - 1) / GB_TN) * ((g.M + GB_TM - 1) / GB_TM) * g.nb1 * g.nb2;
  const int ktiles = (g.K + GB_TK - 1) / GB_TK;
  int s = 1;
  while (tiles * s < (long long)waves * nsm && ktiles / (2 * s) >= min_ktiles) s *= 2;
  return s;
}

// kernel variant (debug / tuning hook): 0 = two-stage static-smem kernel,
// 1 = 3-stage TK 16, 2 = 2-stage TK 32, 3 = 3-stage TK 32, 4 = 4-stage TK 16
static int g_bgemm_variant = 1;

template <int STAGES, int TK, bool AK, bool BK>
static inline void bgemm_pipe_launch_k(dim3 grid, const BGemm& h, cudaStream_t st) {
  constexpr int LDK = TK + 4;
  const size_t smem = sizeof(double) * STAGES * ((AK ? GB_TM * LDK : TK * GB_LD) + (BK ? GB_TN * LDK : TK * GB_LD));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(bgemm_pipe_kernel<STAGES, TK, AK, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  bgemm_pipe_kernel<STAGES, TK, AK, BK><<<grid, 128, smem, st>>>(h);
}

// K-contiguous operands (stride 1 along K, not along M / N) take the [i][k] layout
static int g_bgemm_klayout = 1;

template <int STAGES, int TK>
static inline void bgemm_pipe_launch(dim3 grid, const BGemm& h, cudaStream_t st) {
  const bool ak = g_bgemm_klayout && h.sAm != 1 && h.sAk == 1;
  const bool bk = g_bgemm_klayout && h.sBn != 1 && h.sBk == 1;
  if (ak && bk) bgemm_pipe_launch_k<STAGES, TK, true, true>(grid, h, st);
  else if (ak) bgemm_pipe_launch_k<STAGES, TK, true, false>(grid, h, st);
  else if (bk) bgemm_pipe_launch_k<STAGES, TK, false, true>(grid, h, st);
  else bgemm_pipe_launch_k<STAGES, TK, false, false>(grid, h, st);
}

static inline cudaError_t bgemm_launch(const BGemm& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.nb1 * g.nb2 <= 0) return cudaSuccess;
  const int ks = (g.ksplit > 1 && g.part) ? g.ksplit : 1;
  BGemm h = g;
  h.ksplit = ks;
  dim3 grid((g.N + GB_TN - 1) / GB_TN, (g.M + GB_TM - 1) / GB_TM, g.nb1 * g.nb2 * ks);
  // two-level K addressing exists in the K-contiguous path of the pipelined kernels only
  const int variant = (g.kinB > 0 && (g_bgemm_variant == 0 || g.sBk != 1 || g.kinB % 32 != 0)) ? 1 : g_bgemm_variant;
  if (g.kinB > 0 && (g.sBk != 1 || g.kinB % 16 != 0)) return cudaErrorInvalidValue;
  switch (variant) {
    case 1: bgemm_pipe_launch<3, 16>(grid, h, st); break;
    case 2: bgemm_pipe_launch<2, 32>(grid, h, st); break;
    case 3: bgemm_pipe_launch<3, 32>(grid, h, st); break;
    case 4: bgemm_pipe_launch<4, 16>(grid, h, st); break;
    default: bgemm_kernel<<<grid, 128, 0, st>>>(h);
  }
  if (ks > 1) {
    const size_t mn = (size_t)g.M * g.N;
    dim3 rg((unsigned)((mn + 255) / 256 < 64 ? (mn + 255) / 256 : 64), g.nb1 * g.nb2);
    bgemm_reduce_kernel<<<rg, 256, 0, st>>>(h);
  }
  return cudaGetLastError();
}

}  // namespace tp
