// Gram-space CP-ALS variant (tp_als_w.cu): shapes and plan shared with the planner in tp_als.cu.
#pragma once
#include "tp_common.cuh"

namespace tp {

constexpr int W_RM = 32;                          // padded fitted rank
constexpr int W_SLAB = 8;                         // target terms (columns of C_k) per CTA
constexpr int W_HAD = W_RM * W_SLAB;              // doubles of one had / C slab
constexpr int W_PIECE = W_HAD + W_RM * W_RM + 8;  // had slab | partial Gram | overlap partial (+ pad)

struct WArgs {
  int d, R, r, sweeps, P;           // P column slabs: slab c = target terms [8 c, 8 c + 8)
  int pair;                         // 1: two CTAs (one cluster) per slab, each half of the K range of its T product
  int q[TP_MAXD];
  long long offV[TP_MAXD], offU[TP_MAXD];
  int tile0[TP_MAXD + 1];           // first 8-row tile of mode k in the final-phase item list
  const double* V;
  double* U;
  const double* W;                  // [d][R][R]   W_k = V_k^T V_k
  double* g0buf;                    // [d][W_RM * W_RM] Grams of the initial guess (tiles dealt to the CTAs)
  double* pieces;                   // [2][d][P][W_PIECE] (sweep parity, mode, producer); all-ones words = not written yet
  double* msum;                     // [2][d][W_RM * W_RM] summed partial Grams of the round (sweep parity, mode)
  int* redo;                        // set to 1: ill-conditioned -> the direct kernel reruns the truncation
  const double* norm_sq;
  double* trace;
  int* info;
  double reg;
  int reg_mode;
  double tol, stall;
  int need_resid;
  double cond_max;
  long long* prof;
  int prof_cta;
};

struct WPlan {
  WArgs a;
  size_t smem, ws, ws_inner;
  int uniform_q;
};

int als_w_plan(int d, const int* q, int R, int r, WPlan& pl);
int als_w_enabled();   // debug hook state (part of the planner's cache key)
// launches the setup GEMMs and the kernel; *redo_out = device flag the fallback launch reads
int als_w_run(const WPlan& plan, const double* V, double* U, int sweeps, double reg, int reg_mode, double tol,
              double stall, double* trace, int* info, void* ws, size_t ws_bytes, cudaStream_t st, long long* prof,
              int prof_cta, const int** redo_out);

}  // namespace tp
