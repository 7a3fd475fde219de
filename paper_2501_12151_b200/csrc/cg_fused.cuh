// Persistent cooperative Jacobi-PCG for one local system (see cg_fused.cu).
#pragma once
#include "common.cuh"

namespace qtt {

struct CGFusedArgs {
  // local operator: phil (lb, lo, lk), Ap = permuted core (m, R1 | lo, n), phir (rb, R1, rk)
  const double* phil;
  int lb, lo, lk;
  const double* Ap;
  int m, n, R1;
  const double* phir;
  int rb, rk;
  // vectors of length dim = lb*m*rb (== lk*n*rk for the symmetric local operator)
  const double* b;
  const double* invd;
  double* x;  // in: x0, out: solution
  double *r, *z, *p, *q;
  // optional composed left operator Bop[X][(m,b),(U,n)] = sum_a phil[X,a,U] A[a,m,n,b]
  // (lb * m*R1 * lk*n doubles, built once per solve by cg_fused_build_bop): when set,
  // steps 1+2 of the matvec become ONE batched GEMM phase (one grid barrier less)
  const double* Bop;
  // scratch
  double* t1;     // lb*lo*n*rk (unused with Bop)
  double* t2;     // lb*m*R1*rk
  double* part3;  // S3*dim split-K partials of step 3
  int S3, kt_per3;
  int tileA, tile3;  // tile shape per phase (cg_fused_plan)
  double* red;  // 4*grid doubles (two partial-sum buffers)
  long long dim;
  double atol;
  int maxiter;
  int xany;
  // outputs (device)
  int* out_iters;
  double* out_rnorm;
  unsigned long long* out_mv_ns;  // accumulated wall ns spent in the local matvecs
  // optional (QTT_DEBUG): wall ns per phase [step1, step2, step3, reduce+p.q, update, p-update]
  unsigned long long* phase_ns;
};

int cg_fused_grid(int device);
void cg_fused_plan(int lb, int m, int rb, int R1, int rk, int grid, int& S3, int& kt_per3, int& tileA,
                   int& tile3);
// flops of one matvec with / without the composed left operator (host-side choice)
double cg_fused_flops(int lb, int lo, int lk, int m, int n, int R1, int rb, int rk, bool composed);
void cg_fused_build_bop(const double* phil, int lb, int lo, int lk, const double* Ap, int m, int n, int R1,
                        double* Bop, cudaStream_t s);
void cg_fused_launch(const CGFusedArgs& a, int grid, cudaStream_t s);

}  // namespace qtt
