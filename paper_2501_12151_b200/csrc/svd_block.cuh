// Multi-CTA dense factorizations for large unfoldings (see svd_block.cu).
#pragma once
#include "linalg.cuh"

namespace qtt {

// Thin SVD in = U diag(s) Vt (rows x cols, k = min(rows, cols); s on device, descending)
// by block one-sided Jacobi over column pairs; any of U.p / Vt.p may be null.
void svd_block_jacobi(Ctx& c, CMatView in, MatView U, double* s, MatView Vt);

// Thin QR with LAPACK's factors (dlarfg signs, dorgqr Q) through the blocked
// Householder kernels; Q (m x k) and/or R (k x n) may be null.
void qr_large(Ctx& c, CMatView in, MatView Q, MatView R);

}  // namespace qtt
