// Persistent cooperative Jacobi-PCG on the TMA tile engine (see cg_tma.cu).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace qtt {

// All CG vectors are held TRANSPOSED, [V][U][n] (the local operator is symmetric,
// so output (Y,X,m) and input (V,U,n) share the layout): with that layout every
// operand of the two matvec GEMMs is contiguous along its contraction index, which
// is what the TMA engine needs.
struct CGTmaArgs {
  CUtensorMap map_bop;   // phase 1 A: Bop [(X,m,b)][(U,n)]
  CUtensorMap map_z;     // phase 1 B: z^T [V][(U,n)] (the CG matvec runs on z)
  CUtensorMap map_x;     // phase 1 B: x^T [V][(U,n)] (initial residual)
  CUtensorMap map_phir;  // phase 2 A: phir [Y][(b,V)], row stride K3p
  CUtensorMap map_t2;    // phase 2 B: t2 [(X,m)][(b,V)], row stride K3p
  int lb, m, R1, lk, n, rb, rk;
  long long K3p;
  int p1_rb, p1_cb, p2_rb, p2_cb;  // fragment-block sizes of the phase regions (cg_tma_plan)
  int p1_nf, p1_dedupe, p2_nf, p2_dedupe;
  int box1_a, box1_b, box2_a, box2_b;
  int p1_frun;       // phase 1: fragment-run dealing (one region per CTA, equal fragment counts)
  int stage_stride;  // ring bytes per stage
  int stages;        // ring depth
  const double* b;     // rhs^T
  const double* invd;  // Jacobi inverse diagonal ^T
  double* x;           // in: x0^T, out: solution^T
  double *r, *z, *p, *q;
  double* t2;     // lb*m*K3p
  double* part3;  // S3 * dim split-K partials of phase 2
  int S3, kt_per3;
  double* red;          // 4 * grid
  long long dim;
  double atol;
  int maxiter;
  int xany;
  int* out_iters;
  double* out_rnorm;
  unsigned long long* out_mv_ns;
  unsigned long long* phase_ns;  // optional: [-, phase1, phase2, red, upd, pupd]
  unsigned long long* cta_ns;    // optional (QTT_DEBUG=2): per-CTA busy ns of phase 1 | phase 2
};

struct CGTmaPlan {
  int p1_rb, p1_cb, p2_rb, p2_cb, S3, kt_per3;
  int p1_nf, p1_dedupe, p2_nf, p2_dedupe;
  int box1_a, box1_b, box2_a, box2_b;  // TMA box rows per operand
  int stage_stride, stages, p1_frun;
};

bool cg_tma_supported(int lk, int n);
int cg_tma_grid(int device);
CGTmaPlan cg_tma_plan(int lb, int m, int R1, int lk, int n, int rb, int rk, int grid);
void cg_tma_launch(const CGTmaArgs& a, int grid, cudaStream_t s);
// out[(v*rows + i)] = in[i*cols + v]  (rows = lk*n, cols = rk): [U][n][V] <-> [V][U][n]
void transpose_2d(const double* in, double* out, long long rows, long long cols, cudaStream_t s);

}  // namespace qtt
