/*
 * libqtt -- C ABI of the B200 (sm_100a) QTT AMEn engine.
 *
 * Drop-in boundary for the hot path of the reference package `ttfem`
 * (/root/reference/pkg/src/ttfem).  The reference has no FFI; its boundary is the
 * Python module API.  Each entry point below names the reference function it
 * replaces (file:line); the Python host (paper_2501_12151_b200/) binds them with
 * ctypes and keeps the reference signatures.  INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - All arrays are row-major float64.  Vector cores (r0, n, r1); operator
 *     cores (R0, m, n, R1); environments phi (bra, op, ket), psi (bra, rhs).
 *   - Functions taking `const double*` host pointers copy in, compute on the
 *     device, and copy results out before returning (inputs never mutated,
 *     SPEC.md:156-157).  `qtt_train` handles own device-resident trains.
 *   - Every function returns a status code; on failure qtt_last_error() holds a
 *     thread-local message.  Codes map to ttfem/errors.py:9-34.
 *   - One CUDA stream per context; contexts are independent (re-entrant per handle).
 */
#ifndef QTT_H_
#define QTT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  QTT_OK = 0,
  QTT_ERR_SHAPE = 1,    /* ShapeMismatchError (errors.py:9)  */
  QTT_ERR_SOLVER = 2,   /* SolverError        (errors.py:29) */
  QTT_ERR_CAPACITY = 3, /* CapacityError      (errors.py:13) -- device OOM */
  QTT_ERR_CUDA = 4,     /* CUDA runtime failure / no device                */
  QTT_ERR_ARG = 5,      /* ValueError: invalid argument                    */
  QTT_ERR_FORMAT = 6    /* FormatError        (errors.py:33) -- bad QTT1 container */
};

typedef struct qtt_ctx qtt_ctx;
typedef struct qtt_train qtt_train;

/* ---- lifecycle -------------------------------------------------------------- */
int qtt_version(void);
const char* qtt_last_error(void);
int qtt_ctx_create(int device, qtt_ctx** out);
int qtt_ctx_destroy(qtt_ctx* ctx);
int qtt_ctx_synchronize(qtt_ctx* ctx);
/* the context's cudaStream_t, as an opaque pointer (for event timing by the host) */
void* qtt_ctx_stream(qtt_ctx* ctx);
/* on & 1: per-kernel CUDA-event timing of K1/K2 inside solves (deferred, no syncs);
 * on & 2: per-phase wall timing (synchronizes at phase boundaries); off by default;
 * qtt_stats.launches is the process-wide count of kernels this library launched */
int qtt_ctx_set_profiling(qtt_ctx* ctx, int on);

typedef struct {
  int64_t launches;
  int64_t k1_calls;
  double k1_flops, k1_ms;
  int64_t env_calls;
  double env_flops, env_ms;
  int64_t cg_iters, cg_solves, chol_solves, svd_calls, qr_calls, sweeps, certifications;
  double k1_timed_flops, env_timed_flops; /* flops of the event-timed launches (profiling) */
  /* wall ms per solver phase when profiling: other, direct solve, CG solve, mixed residuals,
   * SVD, QR, environment updates, certification, env pre-pass, local rhs */
  double phase_ms[10];
} qtt_stats;
int qtt_ctx_get_stats(qtt_ctx* ctx, qtt_stats* out);
/* write 256 MiB of scratch on the context stream (evicts the 126 MB L2 between timed steps) */
int qtt_ctx_flush_l2(qtt_ctx* ctx);
/* process-wide number of kernels this library has launched */
int64_t qtt_launch_count(void);
int qtt_ctx_reset_stats(qtt_ctx* ctx);
/* per-local-solve trace of the last solves: 11 int32 per record
 * (sweep, core, r_left, mode, r_right, z_left, z_right, R_left, R_right, path 0=direct/1=cg, cg_iters);
 * *n receives the record count, at most cap records are written */
int qtt_ctx_trace(qtt_ctx* ctx, int32_t* out, int64_t cap, int64_t* n);

/* ---- interface contractions (amen.py:102-160), host buffers ------------------- */
/* y[X,m,Y] = phil[X,a,U] x[U,n,V] A[a,m,n,b] phir[Y,b,V]     replaces _local_matvec  amen.py:134 */
int qtt_local_matvec(qtt_ctx* ctx, const double* phil, const double* A, const double* phir,
                     const double* x, int rX, int Ra, int rU, int m, int n, int Rb, int rY, int rV,
                     double* y);
/* out[U,B,Z] = phi[X,A,Y] ket[Y,n,Z] A[A,m,n,B] bra[X,m,U]   replaces _phi_left_step  amen.py:108 */
int qtt_env_left(qtt_ctx* ctx, const double* phi, const double* bra, const double* A,
                 const double* ket, int rX, int RA, int rY, int m, int n, int RB, int rU, int rZ,
                 double* out);
/* out[B,a,Y] = phi[X,A,Z] ket[Y,n,Z] A[a,m,n,A] bra[B,m,X]   replaces _phi_right_step amen.py:114 */
int qtt_env_right(qtt_ctx* ctx, const double* phi, const double* bra, const double* A,
                  const double* ket, int rX, int RA, int rZ, int m, int n, int Ra, int rB, int rY,
                  double* out);
/* out[U,G] = psi[X,F] f[F,m,G] bra[X,m,U]                    replaces _psi_left_step  amen.py:120 */
int qtt_psi_left(qtt_ctx* ctx, const double* psi, const double* bra, const double* f, int rX,
                 int rF, int m, int rU, int rG, double* out);
/* out[U,F] = psi[X,G] f[F,m,G] bra[U,m,X]                    replaces _psi_right_step amen.py:125 */
int qtt_psi_right(qtt_ctx* ctx, const double* psi, const double* bra, const double* f, int rX,
                  int rG, int rU, int m, int rF, double* out);
/* out[X,m,Y] = psil[X,F] f[F,m,G] psir[Y,G]                   replaces _local_rhs      amen.py:130 */
int qtt_local_rhs(qtt_ctx* ctx, const double* psil, const double* f, const double* psir, int rX,
                  int rF, int m, int rG, int rY, double* out);
/* dense (X,m,Y)x(U,n,V) local matrix                           replaces _local_dense    amen.py:140 */
int qtt_local_dense(qtt_ctx* ctx, const double* phil, const double* A, const double* phir, int rX,
                    int Ra, int rU, int m, int n, int Rb, int rY, int rV, double* out);
/* diagonal of the local matrix                                 replaces _local_diag     amen.py:147 */
int qtt_local_diag(qtt_ctx* ctx, const double* phil, const double* A, const double* phir, int rX,
                   int Ra, int m, int Rb, int rY, double* out);
/* local_rhs(psil,f,psir) - local_matvec(phil,A,phir,u)          replaces _mixed_residual amen.py:154 */
int qtt_mixed_residual(qtt_ctx* ctx, const double* psil, const double* f, const double* psir,
                       const double* phil, const double* A, const double* u, const double* phir,
                       int rX, int rF, int rG, int rY, int Ra, int rU, int m, int n, int Rb, int rV,
                       double* out);

/* ---- device-resident trains ------------------------------------------------ */
/* Upload a train: core_ndim 3 (vector cores r0,n,r1) or 4 (operator cores R0,m,n,R1);
 * shape holds order*core_ndim entries; data the row-major cores back to back.
 * Replaces the TensorTrain / TTLinearOperator constructors (tt.py:110-189). */
int qtt_train_upload(qtt_ctx* ctx, int order, int core_ndim, const int64_t* shape,
                     const double* data, qtt_train** out);
int qtt_train_info(const qtt_train* t, int* order, int* core_ndim, int64_t* numel);
int qtt_train_shape(const qtt_train* t, int64_t* shape);
int qtt_train_download(qtt_ctx* ctx, const qtt_train* t, double* data);
int qtt_train_free(qtt_train* t);
/* QTT1 container (serialize.py:1-101; byte layout serialize.py:3-16) read straight into /
 * written from a device-resident train.  is_operator (out) = 1 for kind 'O'.  Errors: the
 * reference's FormatError cases (bad magic, unknown kind, truncated header / values,
 * trailing bytes) -> QTT_ERR_FORMAT; rank chaining -> QTT_ERR_SHAPE. */
int qtt_train_load_qtt1(qtt_ctx* ctx, const char* path, int* is_operator, qtt_train** out);  /* serialize.py:52 load_tt */
int qtt_train_save_qtt1(qtt_ctx* ctx, const qtt_train* t, const char* path);                 /* serialize.py:33 save_tt */

/* ---- TT algebra (tt.py) ----------------------------------------------------- */
int qtt_orthogonalize_rl(qtt_ctx* ctx, const qtt_train* a, qtt_train** out); /* tt.py:396 */
int qtt_tt_norm(qtt_ctx* ctx, const qtt_train* a, double* out);               /* tt.py:362 */
int qtt_tt_dot(qtt_ctx* ctx, const qtt_train* a, const qtt_train* b, double* out); /* tt.py:351 */
/* max_rank <= 0 means uncapped; operators are rounded over fused (m,n) modes */
int qtt_tt_round(qtt_ctx* ctx, const qtt_train* a, double rel_tol, int max_rank,
                 qtt_train** out);                                            /* tt.py:409, 506 */
int qtt_tt_apply(qtt_ctx* ctx, const qtt_train* A, const qtt_train* x,
                 qtt_train** out);                                            /* tt.py:434 (policy=None) */
/* Dense bridges (tt.py:276-298).  qtt_tt_entries: count entries at multi-indices idx
 * (host int32, count x order, row-major) -> out (host, count doubles); the product of core
 * slices left to right, as tt_entry.  qtt_tt_to_dense: the full C-order (big-endian mode)
 * vector, prod(dims) doubles -> out (host); the reference caps it at 2^22 entries. */
int qtt_tt_entries(qtt_ctx* ctx, const qtt_train* t, const int32_t* idx, int64_t count, double* out); /* tt.py:286 */
int qtt_tt_to_dense(qtt_ctx* ctx, const qtt_train* t, int64_t total, double* out);                    /* tt.py:276 */
/* Config-4 microbench: right-environment pre-pass (amen.py:300-321,
 * _phi_right_step amen.py:114 with bra = ket = x), then one left-to-right sweep of
 * _local_matvec(phi_L[k], A_k, phi_R[k+1], x_k) (amen.py:134) and
 * _phi_left_step(phi_L[k], x_k, A_k, x_k) (amen.py:108).  y_out (optional) receives the
 * local matvec outputs y_k (r_{k-1}, m_k, r_k) as a train.  times (optional, 7 doubles):
 * pre-pass ms, sweep ms, K1 ms, K2 ms (split_timing != 0 only), K1 flops, K2 flops,
 * pre-pass flops. */
int qtt_matvec_sweep(qtt_ctx* ctx, const qtt_train* A, const qtt_train* x, int split_timing,
                     qtt_train** y_out, double* times);
/* ||Ax - f|| / ||f||.  method 0: the reference's QR-sweep norm of the difference train
 * (Kronecker-structured cores + blocked Householder QR); method 1: diagnostic Gram
 * estimate (fast, loses digits when ||A|| ||x|| >> ||Ax - f||). */
int qtt_residual_norm(qtt_ctx* ctx, const qtt_train* A, const qtt_train* x, const qtt_train* f,
                      int method, double* out, int* used_gram);              /* amen.py:87 */

/* ---- dense factorizations of the sweep, host buffers --------------------------- */
/* thin QR, numpy.linalg.qr conventions: q (rows x k), r (k x cols), k = min(rows, cols) */
int qtt_qr(qtt_ctx* ctx, const double* mat, int rows, int cols, double* q, double* r);
/* thin SVD: u (rows x k), s (k, descending), vt (k x cols)   (np.linalg.svd, tt.py:376) */
int qtt_svd(qtt_ctx* ctx, const double* mat, int rows, int cols, double* u, double* s, double* vt);
int qtt_rank_for_tolerance(const double* s, int n, double delta, int* out);  /* tt.py:386 */
/* one local solve (amen.py:170): phil (rl,R0,rl), A (R0,m,m,R1), phir (rr,R1,rr),
 * rhs/prev (rl,m,rr).  Direct (dense + Cholesky) or Jacobi-PCG per the reference rule. */
int qtt_local_solve(qtt_ctx* ctx, const double* phil, const double* A, const double* phir,
                    const double* rhs, const double* prev, int rl, int R0, int m, int R1, int rr,
                    int iterative, int direct_dim_cap, double residual_tol, int iter_cap,
                    int fused_cg, double* u, double* lam, int* iterations);

/* ---- the solve (amen.py:394-510) --------------------------------------------- */
typedef struct {
  double residual_tol;    /* AmenConfig.residual_tol     (amen.py:53) */
  int max_sweeps;         /* AmenConfig.max_sweeps       (amen.py:54) */
  int enrichment_rank;    /* AmenConfig.enrichment_rank  (amen.py:55) */
  int local_iterative;    /* local_solver == "iterative" (amen.py:56) */
  int direct_dim_cap;     /* (amen.py:57) */
  int local_iter_cap;     /* (amen.py:58) */
  double round_tol;       /* rounding.rel_tolerance      (amen.py:59) */
  int round_max_rank;     /* rounding.max_rank, <= 0: None */
  int stagnation_strikes; /* (amen.py:64) */
  int fused_cg;           /* 1: persistent cooperative CG kernel per local solve; 0: per-step launches */
} qtt_amen_params;

typedef struct {
  int converged;
  int sweeps_used;
  double final_relative_residual;
  int certifications_gram, certifications_exact;
  int64_t draws_used;
} qtt_amen_report;

/* draws: the numpy default_rng(seed).standard_normal stream in the reference's
 * consumption order (probe vectors, then z cores, then z redraws); rank_hist has
 * room for max_sweeps*(order+1) ints and res_hist for max_sweeps doubles. */
int qtt_amen_solve(qtt_ctx* ctx, const qtt_train* A, const qtt_train* f, const qtt_train* x0,
                   const qtt_amen_params* prm, const double* draws, int64_t n_draws,
                   qtt_train** x_out, qtt_amen_report* rep, int32_t* rank_hist, double* res_hist);

/* tt_apply (tt.py:434-449, policy=None) into a preallocated train y whose cores have the
 * product's shapes (e.g. a previous qtt_tt_apply result): the Kronecker cores only, no allocation. */
int qtt_tt_apply_into(qtt_ctx* ctx, const qtt_train* A, const qtt_train* x, qtt_train* y);

/* TT-cross (cross.py): maxvol_select (cross.py:80-115) on a tall rows x cols matrix, with the
 * interpolation factor B = A A[piv]^-1 of the chosen rows (cross.py:202-204).  With qr != 0
 * the matrix is first replaced by the Q factor of its thin Householder QR (the
 * np.linalg.qr(mat) of cross.py:220, 245).  piv receives cols row indices, b rows x cols
 * doubles (may be null), *status: 0 dominance reached, 1 rank-deficient input (pivoted-QR rows),
 * 2 singular pivot block (pivoted-QR rows), 3 swap cap reached; | 4 if A[piv] is singular. */
int qtt_maxvol(qtt_ctx* ctx, const double* mat, int rows, int cols, int qr, double tol, int max_iters,
               int32_t* piv, double* b, int* status);

/* One core step of the sweep (amen.py:324-390, the per-core body of _sweep) run by the
 * engine's own per-core code on injected state -- the state-injected parity check at the
 * headline shape.  in[0..10] are host arrays with dims in_dims[3i..3i+2]: x_k, x_nb, z_k
 * (vector cores), phi_k, phi_k1, phiz_k, phiz_k1 (bra, op, ket), psi_k, psi_k1, psiz_k,
 * psiz_k1 (bra, rhs, 1); nb = k+1 when forward, k-1 otherwise (amen.py:356-390).  lam_max is
 * the running spectral bound before the step and f_norm = ||f|| (amen.py:330-337).  *out is
 * a bundle of 7 unchained vector "cores" (read with qtt_train_shape / qtt_train_download):
 * the new x_k, x_nb, z_k and phi, phiz, psi, psiz at the bond the step rebuilt; lam is the
 * step's spectral estimate, rank the truncation rank of _truncated_factor (amen.py:217-234),
 * iters the local CG iterations (0 on the direct path). */
int qtt_amen_step(qtt_ctx* ctx, const qtt_train* A, const qtt_train* f, const qtt_amen_params* prm,
                  int sweep, int k, int forward, double lam_max, double f_norm, int n_in,
                  const double* const* in, const int64_t* in_dims, qtt_train** out, double* lam,
                  int* rank, int* iters);

#ifdef __cplusplus
}
#endif
#endif /* QTT_H_ */
