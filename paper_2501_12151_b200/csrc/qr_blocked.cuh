// Blocked Householder QR for large matrices (see qr_blocked.cu).
#pragma once
#include "engine.cuh"

namespace qtt {

// In-place QR of the column-major m x n matrix W (leading dimension m): on exit the
// upper triangle holds R (dlarfg signs), the strict lower part the reflectors,
// tau[min(m,n)] their scalars -- the LAPACK dgeqrf layout.
void geqrf_blocked(Ctx& c, double* W, int m, int n, double* tau);

// dorgqr: Q (m x k, column-major, leading dimension m) = the first k columns of
// H_1 ... H_k from geqrf_blocked's reflectors (W, tau) -- LAPACK's Q, same signs.
void orgqr_blocked(Ctx& c, const double* W, int m, int k, const double* tau, double* Q);

}  // namespace qtt
