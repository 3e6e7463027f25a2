/*
 * tpde_b200.h -- C ABI of the B200 (sm_100a) rank-truncation hot path.
 *
 * Drop-in boundary for the reference package `tensorpde` (pure Python,
 * /root/reference/pkg/src/tensorpde).  The reference has no FFI; its boundary
 * is the Python API.  Each entry point below replaces the
 * compute behind one reference function; the Python package
 * `paper_1803_10270_b200` binds them through ctypes with the same names,
 * argument meaning and exceptions as the reference.
 *
 * Conventions
 *  - All tensors are real fp64 in DEVICE memory, caller-owned.
 *  - A d-mode CP tensor of rank R is ONE buffer: mode k is the row-major
 *    (Q_k x R) block at element offset R * sum_{k'<k} Q_k'.  Slice k is
 *    exactly the reference's `factors[k]` array (cp.py:43-59).
 *  - `q` arguments are HOST arrays of d mode sizes.
 *  - `stream` is a cudaStream_t passed as void* (no CUDA types in the ABI).
 *  - Scratch comes from a caller-provided device workspace; query its size
 *    with the matching *_ws_bytes function.  The library never allocates.
 *  - Every call returns a status (TP_OK == 0).  Calls are stream-ordered and
 *    re-entrant per stream; results are bitwise deterministic for a fixed
 *    launch configuration.
 */
#ifndef TPDE_B200_H
#define TPDE_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum tp_status {
  TP_OK = 0,
  TP_EINVAL = 1,        /* -> ValueError */
  TP_ENONFINITE = 2,    /* -> ConditioningError / StepFailure (cp.py:178-179, implicit.py:162-163) */
  TP_ENOTPD = 3,        /* Cholesky pivot <= 0 -> ConditioningError */
  TP_ECUDA = 4,         /* -> RuntimeError */
  TP_EWORKSPACE = 5,    /* workspace too small -> RuntimeError */
  TP_EUNSUPPORTED = 6   /* size outside the compiled kernel limits -> ValueError */
};

const char* tp_version(void);
const char* tp_status_string(int status);
/* last CUDA error string seen by the library on this thread (for TP_ECUDA) */
const char* tp_last_error(void);
/* number of SMs of the current device, 0 if none */
int tp_device_sms(void);

/* ---------------------------------------------------------------------------
 * Inner product of two CP tensors.
 * Replaces cp.inner_product / cp.norm (cp.py:111-126) and the target
 * self-norm of _CPTarget (cp.py:186-188):
 *     out = sum_{l<ra, m<rb} prod_k (A_k^T B_k)[l, m]
 * `same` != 0 declares A == B (same buffer): only upper tiles are computed.
 * `out` is a device scalar.
 * ------------------------------------------------------------------------- */
size_t tp_cp_inner_ws_bytes(int d, const int* q, int ra, int rb);
int tp_cp_inner_f64(int d, const int* q, int ra, const double* A, int rb, const double* B,
                    int same, double* out, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Fixed-target Gauss-Seidel CP-ALS (cp.cp_approx_als, cp.py:266-334, with
 * _CPTarget cp.py:183-209 and _solve_gram cp.py:169-180).
 *   V      : target, rank R (device, CP layout)
 *   U      : rank-r guess: initial guess on entry, fit on exit (device, CP layout)
 *   reg    : lambda.  reg_mode 0: fixed lambda = reg.
 *            reg_mode 1: reference rule lambda = reg * max(tr(H),0)/r (cp.py:172)
 *   tol, stall : reference stopping rules (cp.py:329-332); stall = -inf and
 *            tol = 0 run exactly `sweeps` sweeps.
 *   trace  : device array of >= sweeps doubles receiving the residual after
 *            each sweep (cp.py:321-328), or NULL.
 *   info   : device int[2]: {status, sweeps_done}.
 *   grid   : CTAs of the persistent kernel (0 = library choice).
 * The target norm ||V||^2 (needed only when trace != NULL or a stopping rule
 * is active) is computed inside the call.
 * ------------------------------------------------------------------------- */
size_t tp_cp_als_ws_bytes(int d, const int* q, int R, int r, int grid);
int tp_cp_als_f64(int d, const int* q, int R, const double* V, int r, double* U,
                  int sweeps, double reg, int reg_mode, double tol, double stall,
                  double* trace, int* info, int grid, void* ws, size_t ws_bytes, void* stream);
/* Launch plan tp_cp_als_f64 would use (no reference counterpart; introspection
 * for benchmarks/tests): out[0] kernel variant (0 = R-slab per CTA, 1 = clusters
 * of row blocks, 2 = one CTA with the problem resident in shared memory),
 * out[1] CTAs, out[2] CTAs per cluster, out[3] shared bytes/CTA. */
int tp_cp_als_plan(int d, const int* q, int R, int r, int grid, int* out);

/* Fused operator apply + truncation (replaces explicit.py:91-93 /
 * 99-103 target assembly + cp.py:266-334 for the one-CTA problems): the ALS target
 *   V = [A | scale * L(w)],  w = [ws0 W0 | ws1 W1]  (ws* on mode 0; W1 may be NULL),
 * L = sum_t w0[t] (x)_k E_{t,k} (w0 already includes `scale`; mat_idx[t*d + k] indexes
 * mat_off, -1 = identity; the matrices Q_k x Q_k row-major in `mats`, device), is formed
 * inside the kernel from A (rank ra), W0/W1 (rank rw) and the matrices -- L w is never
 * written to memory.  Bitwise equal to materialising the target with tp_cp_apply_f64 and
 * calling tp_cp_als_f64 with tol = 0, stall = -inf, trace = NULL.  Returns
 * TP_EUNSUPPORTED when the problem does not fit the one-CTA kernel. */
int tp_cp_als_recipe_f64(int d, const int* q, int r, const double* A, int ra, const double* W0, double ws0,
                         const double* W1, double ws1, int rw, int n_terms, const double* w0, const int* mat_idx,
                         const double* mats, const long long* mat_off, int n_mats, double* U, int sweeps, double reg,
                         int reg_mode, int* info, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Input-rank-sharded CP-ALS mode steps (BASELINE cfg1 multi-GPU).
 * A rank holds the target slab V (rank R_l = its share of the R input terms,
 * CP layout), the replicated guess U (rank r), its cross slab C (d x r x R_l)
 * and the replicated Grams G (d x r x r).  Per mode update j (cp.py:310-320):
 *   tp_als_shard_rhs_f64    rhs (r x Q_j) = (prod_{k!=j} C_k) V_j^T over the slab
 *   <allreduce rhs across ranks>
 *   tp_als_shard_update_f64 U_j = (A_j^-1 rhs)^T, G_j, C_j[:, slab]
 * ------------------------------------------------------------------------- */
size_t tp_als_shard_ws_bytes(int d, const int* q, int Rl, int r);
int tp_als_shard_init_f64(int d, const int* q, int Rl, const double* V, int r, const double* U, double* C,
                          double* G, void* stream);
int tp_als_shard_rhs_f64(int d, const int* q, int Rl, const double* V, int r, const double* C, int j,
                         double* rhs, void* ws, size_t ws_bytes, void* stream);
int tp_als_shard_update_f64(int d, const int* q, int Rl, const double* V, int r, double* U, double* C, double* G,
                            int j, const double* rhs, double reg, int reg_mode, int* info, void* ws,
                            size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Weight contractions (SURVEY 8(f) f3 device diagnostics): for weight sets
 * W[w] = (W[w][0] | ... | W[w][d-1]) of length sum_k Q_k,
 *   out[w] = sum_l prod_k W[w][k] . F_k[:, l]
 * cp.evaluate (cp.py:84-95: W = basis values at a point) and the moment
 * contractions of diagnostics.moments (diagnostics.py:60-64: W = integration
 * weights).  W and out are device arrays.
 * ------------------------------------------------------------------------- */
int tp_cp_contract_f64(int d, const int* q, int R, const double* F, int nw, const double* W, double* out,
                       void* stream);

/* ---------------------------------------------------------------------------
 * Separable operator apply + concatenation (operators.apply,
 * operators.py:48-62; cp.add/scale, cp.py:98-108).
 * For each term t (0..n_terms-1) and mode k, writes
 *     out_k[:, col_off + t*r_in : col_off + (t+1)*r_in] =
 *         (k == 0 ? scale * weights[t] : 1) * E_{t,k} @ F_k
 * where E_{t,k} is the identity when mat_idx[t*d + k] < 0, else the dense
 * row-major (Q_k x Q_k) matrix at element offset mat_off[mat_idx[t*d+k]] of
 * `mats` (device).  F has rank r_in, out has rank R_out.  Host arrays:
 * q, weights, mat_idx, mat_off.  Terms are written term-major like the
 * reference.
 * ------------------------------------------------------------------------- */
int tp_cp_apply_f64(int d, const int* q, int r_in, const double* F, int n_terms,
                    const double* weights, double scale, const int* mat_idx,
                    const double* mats, const long long* mat_off, int n_mats,
                    double* out, int R_out, int col_off, void* stream);

/* ---------------------------------------------------------------------------
 * Complex128 CP path (the reference's own arithmetic,
 * cp.py:59, and its complex Fourier Galerkin factor matrices, basis.py:168-187).
 * Complex arrays are interleaved (re, im) doubles (numpy/torch complex128
 * layout); sizes count complex elements.
 *   tp_cp_apply_c128 : operators.apply / cp.add / cp.scale (operators.py:48-62,
 *                      cp.py:98-108) with complex weights (host, 2 doubles per
 *                      term), complex scale and complex factor matrices.
 *   tp_cp_inner_c128 : cp.inner_product (cp.py:111-121), conjugate on A;
 *                      out = 2 device doubles (re, im).
 *   tp_cp_als_c128   : cp.cp_approx_als (cp.py:266-334) with the reference's
 *                      normal equations (gram X = had @ T_j^T, factor = X^T),
 *                      one CTA, problem resident in shared memory
 *                      (TP_EUNSUPPORTED when it does not fit).
 * ------------------------------------------------------------------------- */
int tp_cp_apply_c128(int d, const int* q, int r_in, const double* F, int n_terms, const double* weights,
                     double scale_re, double scale_im, const int* mat_idx, const double* mats,
                     const long long* mat_off, int n_mats, double* out, int R_out, int col_off, void* stream);
size_t tp_cp_inner_c128_ws_bytes(int d, const int* q, int ra, int rb);
int tp_cp_inner_c128(int d, const int* q, int ra, const double* A, int rb, const double* B, double* out,
                     void* ws, size_t ws_bytes, void* stream);
size_t tp_cp_als_c128_ws_bytes(int d, const int* q, int R, int r);
int tp_cp_als_c128(int d, const int* q, int R, const double* V, int r, double* U, int sweeps, double reg,
                   int reg_mode, double tol, double stall, double* trace, int* info, void* ws, size_t ws_bytes,
                   void* stream);

/* ---------------------------------------------------------------------------
 * Batched hierarchical-Tucker truncation by hSVD (ht.truncate, ht.py:313-372,
 * with ht.orthogonalize ht.py:294-310) on a balanced binary dimension tree
 * (ht.balanced_tree, ht.py:79-98) with uniform leaf size Q and uniform input
 * rank k at every non-root node.  Batch of `nb` independent tensors.
 *   frames    : device, nb x n_leaves x (Q x k) row-major, leaves in tree preorder
 *   transfers : device, nb x n_interior x (k x k x k) (root: k x k x 1 stored in a
 *               k*k*k slot, only the first k*k entries used), interior nodes in
 *               tree preorder, B[a][b][i] row-major.
 *   Outputs (same layouts with rank r_out = min(r_max, k)):
 *   out_frames nb x n_leaves x (Q x r_out), out_transfers nb x n_interior x
 *   (r_out^3), out_ranks nb x n_nodes ints (kept rank per node),
 *   est nb doubles (sqrt of discarded eigenvalue mass, ht.py:371-372),
 *   norms nb doubles (||h||, ht.py:279-282).
 * eps is the relative tolerance; budget (eps*||h||)^2/(2d-3) per node.
 * ------------------------------------------------------------------------- */
size_t tp_ht_truncate_ws_bytes(int d, int Q, int k, int nb);
int tp_ht_truncate_f64(int d, int Q, int k, int nb, const double* frames, const double* transfers,
                       int r_max, double eps, double* out_frames, double* out_transfers,
                       int* out_ranks, double* est, double* norms,
                       void* ws, size_t ws_bytes, void* stream);
/* Any binary dimension tree (ht.py:55-76 DimensionTree): n_nodes nodes in the
 * caller's order with nodes[0] the root, given as host arrays parent/left/right
 * (-1 = none); frames are packed in leaf order, transfers in interior-node order
 * (node order), the root's k x k x 1 transfer in the first k*k entries of its slot.
 * Same outputs as tp_ht_truncate_f64 (which is this call on balanced_tree(d)). */
size_t tp_ht_truncate_tree_ws_bytes(int n_nodes, const int* parent, const int* left, const int* right, int Q, int k,
                                    int nb);
int tp_ht_truncate_tree_f64(int n_nodes, const int* parent, const int* left, const int* right, int Q, int k, int nb,
                            const double* frames, const double* transfers, int r_max, double eps,
                            double* out_frames, double* out_transfers, int* out_ranks, double* est, double* norms,
                            void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Fixed-rank implicit ALS step (implicit.step, implicit.py:222-301) for an
 * operator pair A = sum_e eta_e (x)_k F_{e,k}, B = sum_z zeta_z (x)_k F_{z,k}
 * with uniform mode size Q.  Replaces build_M (implicit.py:125-131),
 * build_gamma (134-153), solve_beta (156-164: LSQR -> direct regularised
 * Cholesky solve of (M_q + lam I) x = gamma_q) and converged (167-177).
 *   tabs    : device, n_tab x (Q x Q): distinct pairing tables
 *   tab_id  : host, d x ra x ra: tab_id[(k*ra + e)*ra + z] = index of
 *             pairs[k][e][z] = F_{e,k}^T F_{z,k} in tabs
 *   KL, KR  : host ra x ra: eta eta^T and eta zeta^T (implicit.py:106-108)
 *   f_old   : device CP (rank r, d blocks Q x r); f_new: device CP in/out
 *             (initial iterate; the step's result on exit)
 *   schedule: 0 Gauss-Seidel, 1 Jacobi; delta_beta damping (implicit.py:281-282)
 *   orientation: 0 corrected normal equations, 1 reference build_gamma
 *             (implicit.py:137-139)
 *   circ_eig: NULL (dense path: assembled (rQ)^2 system, blocked Cholesky) or,
 *             when every table is circulant, device n_tab x Q x 2 eigenvalues
 *             lambda_t(k) = sum_m tabs[t][m][0] e^{-2 pi i m k/Q}: the system is
 *             solved per DFT frequency (Q Hermitian r x r solves), same minimiser
 *   eps_conv: device double (last sweep's largest relative update)
 *   info    : device int[2] {status bits, sweeps done}
 *   forcing : NULL, or the device CP source term c (rank rf, d blocks Q x rf):
 *             gamma_q += sum_e fcoef[e] (prod_{k!=q} b_k^T S_{k,e} c_k) (S_{q,e} c_q)^T
 *             (implicit.py:140-152), fcoef host ra doubles = dt eta_e; the source
 *             tables S_{k,e} = pairs[k][e][0] (term 0 is the identity in every mode,
 *             the CrankNicolsonPair layout, operators.py:148-150)
 *   eps_tol : the reference loop condition (implicit.py:244) runs on the device:
 *             the sweep whose update reaches eps_tol stops the step (later kernels
 *             of the call are no-ops); no host synchronisation anywhere
 * ------------------------------------------------------------------------- */
size_t tp_implicit_ws_bytes(int d, int Q, int r, int n_tab, int ra, int rf);
int tp_implicit_step_f64(int d, int Q, int r, int ra, int n_tab, const double* tabs, const int* tab_id,
                         const double* KL, const double* KR, const double* f_old, double* f_new,
                         int sweeps, int schedule, double delta_beta, double eps_tol, double lam,
                         int orientation, const double* circ_eig, const double* forcing, int rf,
                         const double* fcoef, double* eps_conv, int* info, void* ws, size_t ws_bytes,
                         void* stream);

/* ---------------------------------------------------------------------------
 * R-sharded fused CP-ALS across GPUs (BASELINE cfg1 multi-GPU, SURVEY 8(e);
 * the per-mode update of cp.py:310-320 with the target's R terms split over
 * `ngpu` ranks).  ONE launch per GPU runs every sweep: each rank forms its
 * R-slab's right-hand-side partials, all ranks exchange them through mapped
 * peer memory (CUDA IPC over NVLink/NVSwitch) after an in-kernel cross-GPU
 * barrier, and every rank reduces them in the same fixed order (rank-major,
 * then cluster), so the replicated fit U is bitwise identical on all ranks.
 * Fixed sweep count (tol = 0, stall = -inf semantics, no trace).
 *   ngroups : groups of CTAs in THIS launch (1 on a real rank; > 1 runs several
 *             ranks' groups co-resident in one launch -- the single-GPU test of
 *             the exchange path); group g is rank rank0 + g
 *   V, U, info, ws : per-group arrays (device pointers): slab (rank R_local,
 *             CP layout), replicated guess/fit (rank r), int[2] status
 *             {bits: 1 not PD, 2 non-finite, 4 peer timeout; sweeps}, workspace
 *   peer    : ngpu device pointers, rank h's exchange buffer as mapped in this
 *             process (tp_als_xg_peer_bytes each, zeroed once at allocation and
 *             reused by every later call of the same ranks and sizes)
 * ------------------------------------------------------------------------- */
size_t tp_als_xg_ws_bytes(int d, const int* q, int R_local, int r, int ngpu, int ngroups);
size_t tp_als_xg_peer_bytes(int d, const int* q, int R_local, int r, int ngpu, int ngroups);
/* out[0] CTAs per rank, out[1] CTAs per cluster, out[2] clusters per rank, out[3] shared bytes */
int tp_als_xg_plan(int d, const int* q, int R_local, int r, int ngpu, int ngroups, int* out);
int tp_als_xg_f64(int d, const int* q, int R_local, int r, int sweeps, double reg, int reg_mode,
                  int ngroups, const double* const* V, double* const* U, int* const* info,
                  void* const* ws, size_t ws_bytes, int ngpu, int rank0, void* const* peer, void* stream);
/* device memory shared between ranks: cudaMalloc'd and zeroed, exported/imported
 * as 64-byte CUDA IPC handles (exchanged by the caller, e.g. all_gather_object) */
int tp_dev_alloc(size_t bytes, void** ptr);
int tp_dev_free(void* ptr);
int tp_ipc_handle(void* ptr, void* handle);
int tp_ipc_open(const void* handle, void** ptr);
int tp_ipc_close(void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* TPDE_B200_H */
