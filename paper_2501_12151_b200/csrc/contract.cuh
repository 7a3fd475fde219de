// Interface (environment) contractions of the AMEn sweep, expressed as chains of
// strided-batched DMMA GEMMs (gemm.cuh).  Layouts follow the reference exactly:
//   phi  at a bond: (bra rank, operator rank, ket rank)          amen.py:104
//   psi  at a bond: (bra rank, rhs rank)                         amen.py:105
//   vector core (r0, n, r1); operator core (R0, m, n, R1)        tt.py:3-8
// The operator core is re-laid out once per upload ("Ap"/"Aq" below) so that
// every contraction step is a plain (batched) GEMM with unit-stride rows.
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace qtt {

// Device scratch arena handed to the contraction chains (stream-ordered).
struct Scratch {
  double* p = nullptr;
  long long n = 0;
};

// Scratch sizes below include the deterministic split-K workspace of the long-K steps.
// Permuted operator-core views (built by permute_op_core):
//   Ap[(m,B),(A,n)] = A[A,m,n,B]   -- left env step and local matvec
//   Aq[(m,a),(A,n)] = A[a,m,n,A]   -- right env step  (same as Ap with R0/R1 roles swapped)
void permute_op_core(const double* A, int R0, int m, int n, int R1, double* Ap, double* Aq,
                     cudaStream_t s);

// phi'[U,B,Z] = sum phi[X,A,Y] ket[Y,n,Z] A[A,m,n,B] bra[X,m,U]        (amen.py:108-111)
long long env_left_scratch(int rX, int RA, int rY, int m, int n, int RB, int rZ, int rU);
void env_left(const double* phi, int rX, int RA, int rY, const double* bra, int rU,
              const double* Ap, int m, int n, int RB, const double* ket, int rZ, double* out,
              Scratch sc, cudaStream_t s);

// phi'[B,a,Y] = sum phi[X,A,Z] ket[Y,n,Z] A[a,m,n,A] bra[B,m,X]        (amen.py:114-117)
long long env_right_scratch(int rX, int RA, int rZ, int m, int n, int Ra, int rY, int rB);
void env_right(const double* phi, int rX, int RA, int rZ, const double* bra, int rB,
               const double* Aq, int m, int n, int Ra, const double* ket, int rY, double* out,
               Scratch sc, cudaStream_t s);

// y[X,m,Y] = alpha * sum phil[X,a,U] v[U,n,V] A[a,m,n,b] phir[Y,b,V] + beta * y   (amen.py:134-137)
long long local_matvec_scratch(int rX, int Ra, int rU, int m, int n, int Rb, int rY, int rV);
void local_matvec(const double* phil, int rX, int Ra, int rU, const double* Ap, int m, int n, int Rb,
                  const double* phir, int rY, int rV, const double* v, double* y, double alpha,
                  double beta, Scratch sc, cudaStream_t s, const int* skip = nullptr);

// psi'[U,G] = sum psi[X,F] f[F,m,G] bra[X,m,U]                          (amen.py:120-122)
void psi_left(const double* psi, int rX, int rF, const double* bra, int m, int rU, const double* f,
              int rG, double* out, Scratch sc, cudaStream_t s);
// psi'[U,F] = sum psi[X,G] f[F,m,G] bra[U,m,X]                          (amen.py:125-127)
void psi_right(const double* psi, int rX, int rG, const double* bra, int rU, int m, const double* f,
               int rF, double* out, Scratch sc, cudaStream_t s);
// b[X,m,Y] = psil[X,F] f[F,m,G] psir[Y,G]                               (amen.py:130-131)
void local_rhs(const double* psil, int rX, int rF, const double* f, int m, int rG, const double* psir,
               int rY, double* out, Scratch sc, cudaStream_t s);

// Dense local matrix  M[(X,m,Y),(U,n,V)]                                 (amen.py:140-144)
long long local_dense_scratch(int rX, int Ra, int rU, int m, int n, int Rb);
void local_dense(const double* phil, int rX, int Ra, int rU, const double* A, int m, int n, int Rb,
                 const double* phir, int rY, int rV, double* mat, Scratch sc, cudaStream_t s);

// diag[X,m,Y] = sum phil[X,a,X] A[a,m,m,b] phir[Y,b,Y]                  (amen.py:147-151)
void local_diag(const double* phil, int rX, int Ra, const double* A, int m, int Rb, const double* phir,
                int rY, double* out, Scratch sc, cudaStream_t s);

// out[c][r] = in[r][c]  (in: rows x cols row-major; out: cols rows with pitch ldo)
void transpose_rows(const double* in, double* out, long long rows, long long cols, long long ldo, cudaStream_t s);

// Flop counts (algorithmic), for the roofline.
double local_matvec_flops(int rX, int Ra, int rU, int m, int n, int Rb, int rY, int rV);
double env_flops(int rX, int RA, int rY, int m, int n, int RB, int rU, int rZ);

}  // namespace qtt
