// Fused direct local solve: Gershgorin bound + Cholesky + both triangular solves
// in one cooperative kernel (see chol_fused.cu).
#pragma once
#include "common.cuh"

namespace qtt {

struct CholArgs {
  double* A;     // dim x dim row-major (ld), overwritten by L in its lower triangle
  int dim;
  long long ld;
  double* x;     // in: right-hand side, out: solution
  double* lam;   // out: max abs row sum (must be zeroed before launch)
  int* info;     // out: 0 or first failing pivot (1-based); must be zeroed before launch
  double* Linv;  // scratch: chol_fused_linv_doubles(dim) -- inverses of the diagonal blocks
  double* y;     // scratch: dim doubles (forward-solve result)
  // optional (QTT_DEBUG): wall ns [row sums, diag factor, panel, trailing, forward, backward]
  unsigned long long* phase_ns;
};

int chol_fused_grid(int device);
long long chol_fused_linv_doubles(int dim);
void chol_fused_launch(const CholArgs& a, int grid, cudaStream_t s);

}  // namespace qtt
