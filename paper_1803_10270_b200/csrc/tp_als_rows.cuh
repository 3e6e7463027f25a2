// Cluster-row CP-ALS variant (tp_als_rows.cu): shapes and plan shared with the
// planner in tp_als.cu.
#pragma once
#include "tp_common.cuh"

namespace tp {

struct RowsArgs {
  int d, R, r, sweeps, S, P;        // S CTAs per cluster (row blocks), P clusters (R-slabs)
  int q[TP_MAXD];
  long long offV[TP_MAXD], offU[TP_MAXD];
  int vrow[TP_MAXD];                // shared-memory row of mode k's V block (rows of ldw doubles)
  int vtot, nb4max, wmax, ldw, kpad, wcol, rs2, gstride, cst_len, piece, ylen;
  int ns;                           // warm-started Newton-Schulz inverse (0: exact sweep every time)
  const double* V;
  double* U;
  double* Y;                        // [2][S][P][ylen] right-hand-side slots (parity of the round)
  unsigned int* flags;              // [2][S][P] round number + 1 once the slot is written
  double* Xw;                       // [CTA][d][RM][pad4(r)] per-CTA warm-start inverses
  double* Hg;                       // [2][P][kpad][pad4(r)] had publish staging (multicast source)
  double* Ag;                       // [2][P][S][gstride] A-block publish staging
  int mc;                           // publishes by TMA multicast from global staging (else st.async)
  int split;                        // rhs product on warps 0-3 while warps 4-7 form A_j and its inverse
  const double* norm_sq;
  double* trace;
  int* info;
  double reg;
  int reg_mode;
  double tol, stall;
  int need_resid;
  long long* prof;
  int prof_cta;
  const int* run_if;                // optional device flag: the launch returns at once unless *run_if != 0
};

struct RowsPlan {
  RowsArgs a;
  int rm;
  size_t smem, ws, ws_inner;
};

int als_rows_plan(int d, const int* q, int R, int r, int S_force, int P_force, RowsPlan& pl);
int als_rows_run(const RowsPlan& plan, const double* V, double* U, int sweeps, double reg, int reg_mode, double tol,
                 double stall, double* trace, int* info, void* ws, size_t ws_bytes, cudaStream_t st, long long* prof,
                 int prof_cta, int ns, const int* run_if = nullptr);

}  // namespace tp
