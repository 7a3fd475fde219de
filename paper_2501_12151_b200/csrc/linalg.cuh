// Dense FP64 building blocks of the sweep: Householder QR (LAPACK dgeqrf/dorgqr
// sign conventions), one-sided Jacobi SVD, blocked Cholesky + triangular solves,
// deterministic reductions and small elementwise kernels.
#pragma once
#include <vector>

#include "common.cuh"
#include "engine.cuh"

namespace qtt {

struct MatView {
  double* p = nullptr;
  int rows = 0, cols = 0;
  long long rs = 0, cs = 0;  // element (i, j) at p[i*rs + j*cs]
};
struct CMatView {
  const double* p = nullptr;
  int rows = 0, cols = 0;
  long long rs = 0, cs = 0;
};
inline MatView rowmajor(double* p, int rows, int cols) { return {p, rows, cols, cols, 1}; }
inline CMatView crowmajor(const double* p, int rows, int cols) { return {p, rows, cols, cols, 1}; }
inline CMatView ctrans(CMatView v) { return {v.p, v.cols, v.rows, v.cs, v.rs}; }
inline MatView trans(MatView v) { return {v.p, v.cols, v.rows, v.cs, v.rs}; }
inline CMatView cview(MatView v) { return {v.p, v.rows, v.cols, v.rs, v.cs}; }

// Thin QR of in (m x n): Q (m x k), R (k x n), k = min(m, n).  Either output may
// have p == nullptr.  Householder reflectors with dlarfg's sign rule, Q formed
// as in dorg2r, so Q and R match numpy.linalg.qr up to rounding.
void qr(Ctx& c, CMatView in, MatView Q, MatView R);
// The single-CTA blocked (compact-WY, DMMA trailing updates) kernel behind qr() for matrices whose
// working set fits one CTA's shared memory (qr_cta.cu); qr_cta_smem_doubles(m, n) is that set.
long long qr_cta_smem_doubles(int m, int n);
void qr_cta(Ctx& c, CMatView in, MatView Q, MatView R);

// Thin SVD of in (m x n), k = min(m, n): U (m x k), s (k, device), Vt (k x n),
// singular values sorted descending.  Householder QR to a k x k triangle, then
// one-sided (Hestenes) Jacobi on it: singular values with high relative accuracy,
// which the rank rule (tt.py:386-393) needs near the truncation threshold.
void svd(Ctx& c, CMatView in, MatView U, double* s, MatView Vt);

// In-place lower Cholesky of the row-major dim x dim matrix (ld) -- blocked,
// right-looking, DMMA trailing updates.  *info (device) = 0 on success, else
// j+1 for the first non-positive pivot (LAPACK dpotrf convention).
void potrf_lower(Ctx& c, double* A, int dim, long long ld, int* info);
// A[i][i] += v for i < n (row-major, leading dimension ld)
void add_diag(Ctx& c, double* A, int n, long long ld, double v);
// Solve (L L^T) x = b in place, L from potrf_lower (dpotrs).
void potrs_lower(Ctx& c, const double* L, int dim, long long ld, double* b);
// *out = max_i sum_j |A[i,j]|   (Gershgorin bound, amen.py:190)
void max_abs_row_sum(Ctx& c, const double* A, int dim, long long ld, double* out);

// Deterministic reductions into a device scalar (fixed grid, fixed order).
void dot(Ctx& c, const double* a, const double* b, long long n, double* out);
void sum(Ctx& c, const double* a, long long n, double* out);
void nrm2(Ctx& c, const double* a, long long n, double* out);  // sqrt(sum a^2)

// Host readback of device scalars (synchronizes the context stream).
void read_scalars(Ctx& c, const double* dev, int n, double* host);

// y[(a,x), m, (b,y)] = sum_n A[a,m,n,b] x[x,n,y]          (tt.py:443-447 Kronecker core)
void kron_core(Ctx& c, const double* A, int Ra0, int m, int n, int Ra1, const double* x, int rx0,
               int rx1, double* y);
// All Kronecker cores of a TT-matvec in one launch: core k reads A_k (Ra0, m, n, Ra1), x_k
// (rx0, n, rx1) and writes y_k ((Ra0 rx0), m, (Ra1 rx1)); row0 is filled in by kron_all.
constexpr int kKronMaxCores = 64;
struct KronDesc {
  const double* A;
  const double* x;
  double* y;
  long long row0;
  int Ra0, m, n, Ra1, rx0, rx1;
};
void kron_all(Ctx& c, const std::vector<KronDesc>& cores);
// out[i*ld_out + j] = scale[i] * in[i*ld_in + j]  (rows scaled), for S V^T style products
void scale_rows(Ctx& c, const double* in, long long ld_in, const double* scale, int rows, int cols,
                double* out, long long ld_out);
// copy a strided view into another view of the same shape
void copy_view(Ctx& c, CMatView in, MatView out);
void fill(Ctx& c, double* p, long long n, double v);
// y = a*x + b*y
void axpby(Ctx& c, long long n, double a, const double* x, double b, double* y);
// diagonal of an operator core: d[a, m, b] = A[a, m, m, b]
void op_core_diag(Ctx& c, const double* A, int R0, int m, int R1, double* d);

}  // namespace qtt
