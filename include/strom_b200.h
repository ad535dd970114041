/*
 * strom_b200 -- C ABI of the B200-native (sm_100a) hot path of arXiv 1910.01260
 * (streaming incremental SVD, per-mode temporal bases, block-structured
 * space-time reduced operator and its solve).
 *
 * Conventions
 *   - plain C types only; every pointer argument named *_dev is DEVICE memory,
 *     *_host is host memory; `stream` is a cudaStream_t passed as void*
 *     (NULL = legacy default stream).  All work is stream-ordered and
 *     asynchronous unless the comment says "synchronizes".
 *   - return value: 0 on success, otherwise a STROM_E* code; the message is
 *     strom_last_error() (thread-local).  The Python mirror maps the codes to
 *     the reference's exception types (ValueError, BasisError,
 *     SingularMatrixError).
 *   - dense matrices are column-major with an explicit leading dimension
 *     unless a parameter says row-major.
 *
 * Each entry point cites the reference interface it replaces (file:line
 * under the reference's pkg/src/strom/).
 */
#ifndef STROM_B200_H
#define STROM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STROM_B200_ABI_VERSION 1

#define STROM_OK 0
#define STROM_EINVAL 1     /* shape / argument error        -> ValueError          */
#define STROM_ECUDA 2      /* CUDA runtime failure                                 */
#define STROM_ENUMERIC 3   /* non-finite input              -> ValueError          */
#define STROM_ESINGULAR 4  /* pivot below floor             -> SingularMatrixError */
#define STROM_ERANK 5      /* rank / ceiling violation      -> BasisError          */
#define STROM_EINTERNAL 6

const char* strom_last_error(void);
int strom_abi_version(void);
int strom_device_synchronize(void);
/* Give back device memory the library keeps for reuse: the spare store block a compaction
 * ping-pongs with (kept only for stores of 1 GiB and more, and only while a state is alive).
 * Call it before a large allocation of your own, e.g. the n x r export of phi at capacity
 * sizes.  No reference counterpart (device memory management). */
void strom_trim_cache(void);

/* Built-in profiling (used by bench.py for the live roofline): per kernel kind
 * (0 proj pass, 1 residual pass, 2 step A, 3 step B, 4 V update, 5 compaction,
 * 6 tall GEMM, 7 spatial, 8 ST Gram, 9 ST small, 10 LU, 11 temporal, 12 other)
 * the launch count, the summed CUDA-event duration (only while enabled) and
 * the algorithmic bytes moved.  strom_profile_read synchronizes the device. */
void strom_profile_enable(int32_t on);
int strom_profile_reset(void);
int strom_profile_read(int32_t nkinds, int64_t* launches_host, double* ms_host, double* bytes_host);
/* Per-launch event durations (ms, launch order) of one kind recorded since the
 * last reset: at most `max` values into ms_host, the total count into n_out.
 * Lets a caller separate launches that returned at once (a pass skipped by a
 * device-side decision moves no bytes) from the ones that did the work. */
int strom_profile_durations(int32_t kind, int32_t max, float* ms_host, int32_t* n_out);

/* fp64 tensor-pipe (DMMA) throughput probe: launches ctas_per_sm x SMs CTAs of
 * `iters` DMMA rounds on `stream`; *flops_out = flops issued (time it with events). */
int strom_fp64_probe(int32_t iters, int32_t ctas_per_sm, void* stream, double* flops_out);

/* ------------------------------------------------------------------------
 * Streaming incremental SVD  (basis.py:30-194, PAPER.md Algorithms 1-2)
 *
 * A strom_isvd is one immutable SvdState (basis.py:30-62).  Updates are
 * functional like the reference's dataclasses.replace (basis.py:127,176): the
 * source handle stays valid; every call returns a new handle that the caller
 * frees with strom_isvd_free.  Decisions (dependent / truncate / drift-QR /
 * restart) are taken on the device; no host round trip per snapshot.
 * ------------------------------------------------------------------------ */
typedef struct strom_isvd strom_isvd;

#define STROM_CAP_RESTART 0
#define STROM_CAP_TRUNCATE 1

/* decision bits of the update that produced a state (strom_isvd_info.flags) */
#define STROM_F_DEPENDENT 1
#define STROM_F_TRUNCATED 2
#define STROM_F_QR 4
#define STROM_F_RESTART 8
#define STROM_F_REJECTED 16

typedef struct {
  int64_t n;          /* rows (spatial DOFs)                              */
  int64_t k;          /* columns ingested (SvdState.k, basis.py:45)       */
  int32_t rank;       /* sigma.size (basis.py:60-62)                      */
  int32_t ncols_u;    /* columns of the append-only store in use          */
  int32_t n_rejected, n_dependent, n_truncated, n_restarts; /* basis.py:50-54 */
  int32_t flags;      /* STROM_F_* of the last update                     */
  int32_t status;     /* 0, or STROM_ENUMERIC after a non-finite column   */
  double last_p;      /* Pythagorean residual norm of the last update     */
  double last_drift;  /* |phi_0 . phi_last| of the last update            */
  double last_xnorm;  /* ||x|| of the last update                         */
  double tol_svd, tol_sv;
  int64_t r_max;      /* -1 = uncapped                                    */
  int32_t cap_mode;   /* STROM_CAP_*                                      */
  int32_t pad;
  double last_p_sq;   /* unclamped x.x - ell.ell of the last update (basis.py:136) */
} strom_isvd_info;

/* isvd_init (basis.py:65-102): start the stream at its k-th column x_dev[n]. */
int strom_isvd_init(int64_t n, const double* x_dev, int64_t k, double tol_svd, double tol_sv,
                    int64_t r_max, int32_t cap_mode, void* stream, strom_isvd** out);

/* isvd_update (basis.py:105-184): fold one column; *out is a new state. */
int strom_isvd_update(strom_isvd* src, const double* x_dev, void* stream, strom_isvd** out);

/* ingest_simulation (basis.py:187-194): fold ncols columns of X (column-major,
 * leading dimension ldx) left to right.  x_on_host != 0: X is host memory
 * (pinned for overlap); the columns are streamed to the device in chunks on a
 * copy stream overlapped with the updates. */
int strom_isvd_ingest(strom_isvd* src, const double* X, int64_t ldx, int64_t ncols, int32_t x_on_host,
                      void* stream, strom_isvd** out);

/* SvdState fields: synchronizes `stream` and reads the device header. */
int strom_isvd_query(strom_isvd* h, void* stream, strom_isvd_info* out);

/* Materialise phi (n x rank, ROW-major like the reference's C-ordered array),
 * sigma (rank) and v (k x rank, row-major).  Any output may be NULL. */
int strom_isvd_export(strom_isvd* h, double* phi_dev, double* sigma_dev, double* v_dev, void* stream);

/* SvdState(phi, sigma, v, k, ...) constructor (basis.py:30-58) from explicit
 * device arrays (phi n x r row-major, v k x r row-major).  phi need not be
 * orthonormal; it must have full column rank (its Gram is Cholesky-factored).
 * counters4 = {n_rejected, n_dependent, n_truncated, n_restarts} (host). */
int strom_isvd_load(int64_t n, int64_t k, int64_t r, const double* phi_dev, const double* sigma_dev,
                    const double* v_dev, double tol_svd, double tol_sv, int64_t r_max, int32_t cap_mode,
                    const int32_t* counters4_host, void* stream, strom_isvd** out);

/* Same state given in factored form phi = U W with U (n x c, column-major,
 * ldu) and W (c x r, column-major, ldw); L (c x c lower, ldl) is the Cholesky
 * factor of U^T U, or NULL when U has orthonormal columns. */
int strom_isvd_load_factored(int64_t n, int64_t k, int64_t c, int64_t r, const double* u_dev, int64_t ldu,
                             const double* w_dev, int64_t ldw, const double* l_dev, int64_t ldl,
                             const double* sigma_dev, const double* v_dev, double tol_svd, double tol_sv,
                             int64_t r_max, int32_t cap_mode, const int32_t* counters4_host, void* stream,
                             strom_isvd** out);

/* The device representation phi = U W (U[:, 0:c] n x c with ld n, W c x r
 * with ld c, L = chol(U^T U) c x c with ld c), for invariant checks.
 * Synchronizes.  Any output may be NULL. */
int strom_isvd_factors(strom_isvd* h, double* u_dev, double* w_dev, double* l_dev, void* stream);

/* ------------------------------------------------------------------------
 * Row-sharded incremental SVD over several GPUs (the reference
 * is single-process -- this is the multi-GPU form of basis.py:105-194).
 *
 * Rank r of a group owns a block of rows of every snapshot and of the left
 * basis; sigma, V and every decision are replicated bit-identically.  The
 * per-rank partial sums of the tall kernels (U^T x, x.x, U^T r, r.r, window
 * projections, compaction Grams) cross the GPUs in ONE small kernel over
 * NVLink peer memory (mailboxes mapped by CUDA IPC; csrc/shard.cuh), summed in
 * rank order on every rank.
 *
 * Set-up (one process per GPU):
 *   1. strom_shard_mailbox_create(world, &g, handle)   on every rank
 *   2. all-gather the 64-byte handles in rank order (torch.distributed / MPI)
 *   3. strom_shard_connect(g, rank, n_global, handles)
 *   4. strom_shard_make_current(g); strom_isvd_init(n_local, x_local, ...) --
 *      a state created while a group is current is that rank's shard; its
 *      successors (update / ingest) inherit the group.  make_current(NULL)
 *      afterwards.  Every rank must issue the same sequence of calls.
 * strom_isvd_export then yields the rank's rows of phi and the replicated
 * sigma and V.  A peer that stops responding makes the exchange time out
 * (STROM_SHARD_TIMEOUT_MS, default 5000) and the next strom_isvd_query fail
 * with STROM_ECUDA instead of hanging the GPU.
 * ------------------------------------------------------------------------ */
typedef struct strom_shard strom_shard;
#define STROM_SHARD_HANDLE_BYTES 64
#define STROM_SHARD_MAX_RANKS 8

int strom_shard_mailbox_create(int32_t world, strom_shard** out, void* handle64_out_host);
int strom_shard_connect(strom_shard* g, int32_t rank, int64_t n_global, const void* handles_host);
/* Single-process group of `world` virtual ranks on the current device (test
 * harness): out[world]; each rank is driven by its own host thread and the
 * exchanges are ordered by stream events, never by kernels waiting on kernels. */
int strom_shard_create_local(int32_t world, int64_t n_global, strom_shard** out);
/* Thread-local: states created by strom_isvd_init / strom_isvd_load* on this
 * thread join group g (NULL: none). */
void strom_shard_make_current(strom_shard* g);
/* Synchronizes the device; exchanges completed and the sticky error word
 * (0 ok, 1 peer timeout, 2 vector too large). */
int strom_shard_status(strom_shard* g, int64_t* exchanges_out, int32_t* error_out);
void strom_shard_free(strom_shard* g);

/* Diagnostics: mean ms of `iters` fused passes over a synthetic n x c store. */
int strom_debug_pass_bw(int64_t n, int32_t c, int32_t iters, int32_t reserve, double* ms_out);

/* Diagnostics: step-B phase timestamps (clock64, 8 slots) into dev_buf; NULL disables. */
void strom_debug_tprobe(long long* dev_buf);
void strom_debug_lu_probe(long long* dev_buf); /* persistent LU: 8 globaltimer stamps per CTA (diagnostics) */
void strom_debug_trace(long long* dev_buf, int64_t rows); /* window-mode iSVD: 16 stamps per update (diagnostics) */

void strom_isvd_free(strom_isvd* h);

/* ------------------------------------------------------------------------
 * Temporal bases  (basis.py:275-302 build_basis_set's per-mode loop)
 * v_dev: the k x r right singular matrix, column-major (ld ldv >= n_mu*n_steps).
 * For every mode i < n_s: T_i = v[:, i] reshaped N_t x n_mu (basis.py:215-228),
 * thin SVD with the reference's sign rule; psi_dev receives the first n_t
 * left vectors as (n_s, N_t, n_t) C-order, ranks_dev (int32 n_s) the rank
 * #{sigma > max(N_t, n_mu) eps sigma_0}, sigma_dev (n_s x min(N_t, n_mu)).
 * The caller raises BasisError when n_t > ranks[i] (basis.py:297-300).
 * ------------------------------------------------------------------------ */
int strom_temporal_bases(const double* v_dev, int64_t ldv, int64_t r, int64_t n_steps, int64_t n_mu,
                         int64_t n_s, int64_t n_t, double* psi_dev, int32_t* ranks_dev, double* sigma_dev,
                         void* stream);

/* ------------------------------------------------------------------------
 * Spatial reduced operators  (spatial.py:45-67 build_spatial_rom)
 * CSR A (indptr n+1, indices, data; index_bits 32 or 64), phi element (i, j)
 * at phi_dev[i*phi_rs + j*phi_cs] (row- or column-major), extra: column-major
 * n x ne (ld ext_ld) right-hand columns, xref: n-vector or NULL.
 * out_dev: row-major ns x q, q = ns + ne + (xref != NULL):
 *   [A_hat | phi^T extra | phi^T (A xref)].   A phi is never materialised.
 * ------------------------------------------------------------------------ */
int strom_spatial_reduce_csr(int64_t n, const void* indptr_dev, const void* indices_dev, const double* data_dev,
                             int32_t index_bits, const double* phi_dev, int64_t phi_rs, int64_t phi_cs,
                             int64_t ns, const double* extra_dev, int64_t ext_ld, int64_t ne,
                             const double* xref_dev, double* out_dev, void* stream);

/* Tiled-ELL operator form (built once per operator, like a sparse library's
 * SpMM preprocessing) and the spatial reduction over it: the fast path for
 * column-major phi with n_s, q <= 64 (same contractions and output as
 * strom_spatial_reduce_csr).  Per 64-row tile: K off-diagonal slots (uint32
 * column, double value) and the diagonal; K in {4, 6, 8, 16} >= max
 * off-diagonal entries per row.  eidx_dev: ceil(n/64) * K * 64 uint32,
 * eval_dev: ceil(n/64) * (K+1) * 64 doubles.  *reach_out (host) = max(col -
 * row) over off-diagonal entries (-1: none), the forward reach used to stream
 * phi rows into L2 ahead of the gathers. */
int strom_csr_to_ell(int64_t n, const void* indptr_dev, const void* indices_dev, const double* data_dev,
                     int32_t index_bits, int32_t K, uint32_t* eidx_dev, double* eval_dev, int64_t* reach_out,
                     void* stream);
int strom_spatial_reduce_ell(int64_t n, int32_t K, const uint32_t* eidx_dev, const double* eval_dev, int64_t reach,
                             const double* phi_dev, int64_t ld, int64_t ns, const double* extra_dev, int64_t ext_ld,
                             int64_t ne, const double* xref_dev, double* out_dev, void* stream);

/* Y = A X for the CSR operator and a row-major X (n_cols(A) x m, leading dimension ldx);
 * Y is n x m row-major (ldy).  The sparse applies of the a-posteriori bounds: A x_k for
 * every step of a trajectory (system.py:249-275) and operator_norm's power iteration on a
 * sparse operator (bounds.py:60-70).  Rows are summed in CSR order. */
int strom_csr_spmm(int64_t n, const void* indptr_dev, const void* indices_dev, const double* data_dev,
                   int32_t index_bits, const double* x_dev, int64_t ldx, int64_t m, double* y_dev, int64_t ldy,
                   void* stream);

/* Dense LU with partial pivoting kept for repeated solves -- the reference's
 * StepSolver pattern (system.py:106-125: one factor per dt, one solve per
 * step).  a_dev / lu_dev: n x n column-major, factored in place; piv_dev: n
 * ints; x_dev: n x nrhs column-major, overwritten.  Asynchronous; no pivot-floor
 * test (strom_dense_solve has it). */
int strom_dense_lu(int64_t n, double* a_dev, int32_t* piv_dev, void* stream);
int strom_dense_lu_solve(int64_t n, const double* lu_dev, const int32_t* piv_dev, double* x_dev, int64_t nrhs,
                         void* stream);

/* fom_march (system.py:150-163) on the device: (I - dt_k A) x_k = x_{k-1} +
 * dt_k B f_k for k = 1..N_t by Jacobi-preconditioned BiCGSTAB (relative
 * residual tol, at most maxit iterations per step) in one cooperative kernel,
 * over A's tiled-ELL form (strom_csr_to_ell).  b_dev: n x m column-major;
 * f_dev: N_t x m row-major (row k = input of step k+1); dt_dev: N_t;
 * states_dev: n x N_t column-major (column k-1 = x_k).  iters_out (host,
 * may be NULL): iterations per step.  A step that misses tol is a numerical
 * error. */
int strom_fom_march(int64_t n, int32_t K, const uint32_t* eidx_dev, const double* eval_dev, const double* b_dev,
                    int64_t m, const double* x0_dev, const double* dt_dev, const double* f_dev, int64_t nt, double tol,
                    int32_t maxit, double* states_dev, int32_t* iters_out, void* stream);

/* The same march for a tridiagonal or periodic tridiagonal A (1-D problems; n <= 4096,
 * n = 2^k when periodic): a direct solve per step by parallel cyclic reduction in one CTA --
 * the reference's StepSolver pattern (system.py:106-125: factor once per dt, solve per step),
 * with the elimination multipliers tabulated per distinct dt.  lo[i] = A(i, i-1), di[i] =
 * A(i, i), up[i] = A(i, i+1); periodic: lo[0] = A(0, n-1), up[n-1] = A(n-1, 0).  No pivoting:
 * the caller checks that I - dt A is strictly diagonally dominant.  v_dev non-null (then
 * b, f, x0 may be null): the block substitution of strom_st_apply_inverse instead. */
int strom_fom_march_tridiag(int64_t n, const double* lo_dev, const double* di_dev, const double* up_dev,
                            int32_t periodic, const double* b_dev, int64_t m, const double* x0_dev,
                            const double* dt_dev, const double* f_dev, const double* v_dev, int64_t nt,
                            double* states_dev, void* stream);

/* (A_st)^{-1} v by forward block substitution (system.py:195-213): x_k solves
 * (I - dt_k A) x_k = x_{k-1} + v_k with x_0 = 0, by the same cooperative
 * BiCGSTAB march as strom_fom_march; v_dev, out_dev: n x N_t column-major.
 * The adjoint (system.py:216-233) is this call on the transposed operator's
 * ELL form with the blocks and steps reversed. */
int strom_st_apply_inverse(int64_t n, int32_t K, const uint32_t* eidx_dev, const double* eval_dev, const double* dt_dev,
                           const double* v_dev, int64_t nt, double tol, int32_t maxit, double* out_dev,
                           int32_t* iters_out, void* stream);

/* Workload generator (bench/test support, not a reference interface): nb
 * columns t0 .. t0+nb-1 of the capacity stream X = Q diag(sigma) W^T + E with
 * an implicit randomized-Hadamard Q (Q[i,c] = s_i (-1)^popcount(i & p_c) /
 * sqrt(n), n = 2^m, never stored) and counter-hash Gaussian noise.
 * coef_dev[c*nb + b] = sigma_c W[t0+b, c]; prow_dev: rank distinct Hadamard
 * rows; out_dev: n x nb column-major (ldo).  nb in {1, 2, 4, 8, 16}. */
int strom_gen_lowrank_batch(int64_t n, int32_t rank, int32_t nb, const double* coef_dev, const int64_t* prow_dev,
                            uint64_t seed, int64_t t0, double noise, double* out_dev, int64_t ldo, void* stream);

/* ------------------------------------------------------------------------
 * Space-time reduced system  (spacetime.py:43-115 build_st_matrix /
 * build_st_input / build_st_init, spacetime.py:128-151 build_st_rom)
 *   ahat n_s x n_s row-major; psi (n_s, N_t, n_t) C-order; dt N_t;
 *   bhat n_s x m row-major; f: m values (constant_input) or N_t x m row-major;
 *   x0hat n_s.  Outputs a_st (NT x NT row-major), f_st, x0_st (NT = n_s n_t,
 *   index j*n_s + i); pass NULL for outputs not wanted (a_st NULL skips the
 *   matrix; f_st and x0_st come together).
 * ------------------------------------------------------------------------ */
int strom_st_assemble(const double* ahat_dev, const double* psi_dev, const double* dt_dev, int64_t nsteps,
                      int64_t ns, int64_t nt, const double* bhat_dev, int64_t m, const double* f_dev,
                      int32_t constant_input, const double* x0hat_dev, double* ast_dev, double* fst_dev,
                      double* x0st_dev, void* stream);

/* reconstruct_states (spacetime.py:180-186; replaces its einsum + phi_s @ coeffs):
 * out (N x nsteps, row-major, ldo) = phi (N x ns, column-major, ldphi) C with
 * C[i, k] = sum_j psi[i, k, j] xhat[j*ns + i]; psi is the (ns, nsteps, nt)
 * temporal stack, xhat the ns*nt space-time solution (index j*ns + i). */
int strom_st_reconstruct(int64_t N, int64_t ns, int64_t nt, int64_t nsteps, const double* phi_dev, int64_t ldphi,
                         const double* psi_dev, const double* xhat_dev, double* out_dev, int64_t ldo, void* stream);

/* ------------------------------------------------------------------------
 * Dense kernels  (linalg.py:41-99)
 * ------------------------------------------------------------------------ */
/* solve_dense: LU with partial pivoting of a (n x n column-major, overwritten)
 * and nrhs right-hand sides x (n x nrhs column-major, overwritten by the
 * solution).  STROM_ESINGULAR with "pivot i" when |U_ii| <= 1e-14 ||a||_F
 * (synchronizes).  piv_dev (int32 n) and info_dev (3 doubles) may be NULL. */
int strom_dense_solve(int64_t n, double* a_dev, double* x_dev, int64_t nrhs, int32_t* piv_dev, double* info_dev,
                      void* stream);

/* qr: thin QR with diag(R) >= 0; m (rows x cols, column-major, ld) <- Q, r_dev <- R (cols x cols). */
int strom_qr(int64_t rows, int64_t cols, double* m_dev, int64_t ld, double* r_dev, void* stream);

/* thin_svd: m (rows x cols column-major) = w diag(s) v^T, sigma descending, the
 * largest-|.| entry of every column of w made >= 0 (linalg.py:31-38).
 * w: rows x kmin, v: cols x kmin (column-major), kmin = min(rows, cols). */
int strom_thin_svd(int64_t rows, int64_t cols, const double* m_dev, double* w_dev, double* s_dev, double* v_dev,
                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STROM_B200_H */
