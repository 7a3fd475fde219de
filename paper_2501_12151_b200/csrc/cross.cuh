// TT-cross building blocks (cross.py): maxvol row selection + interpolation factor.
#pragma once
#include "common.cuh"
#include "engine.cuh"

namespace qtt {

// Rows of the tall N x r row-major device matrix A forming a quasi-dominant r x r submatrix
// (cross.py:80-115): rows_dev[r] and B = A A[rows]^-1 (N x r, device).  Returns the status:
// 0 dominance reached, 1 rank-deficient input (pivoted-QR rows kept), 2 singular pivot block
// (pivoted-QR rows kept), 3 swap cap reached; | 4 when A[rows] itself is singular (B unset).
int maxvol(Ctx& c, const double* A, int N, int r, double tol, int max_iters, double* B, int* rows_dev,
           int* status_dev);

}  // namespace qtt
