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
  QTT_ERR_ARG = 5       /* ValueError: invalid argument                    */
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
/* per-kernel CUDA-event timing of K1/K2 inside solves (off by default) */
int qtt_ctx_set_profiling(qtt_ctx* ctx, int on);

typedef struct {
  int64_t launches;
  int64_t k1_calls;
  double k1_flops, k1_ms;
  int64_t env_calls;
  double env_flops, env_ms;
  int64_t cg_iters, cg_solves, chol_solves, svd_calls, qr_calls, sweeps, certifications;
} qtt_stats;
int qtt_ctx_get_stats(qtt_ctx* ctx, qtt_stats* out);
int qtt_ctx_reset_stats(qtt_ctx* ctx);

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

#ifdef __cplusplus
}
#endif
#endif /* QTT_H_ */
