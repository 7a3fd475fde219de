// TT-cross building blocks on the device (cross.py:80-115, 202-265): the maxvol row selection
// of a tall matrix and the interpolation factor Q Q[piv]^-1 of a cross half-sweep.
//
// One CTA per matrix (the cross sweeps factor small rk*n x r unfoldings, r <= max_rank), the
// matrix and its scratch in global memory (L1/L2-resident at these sizes):
//   1. pivoted rows: greedy largest-residual row, the rest orthogonalised against it -- the
//      column-pivoted QR of A^T that cross.py:94 asks scipy for (ties: lowest index, as LAPACK's
//      idamax), |R_kk| = the residual norm of pivot k;
//   2. maxvol swaps: B = A A[rows]^-1 (Gauss-Jordan inverse with partial pivoting), the
//      entry of largest magnitude (first in row-major order, as np.argmax) swapped in while it
//      exceeds 1 + tol (cross.py:103-113);
// and B of the final rows is returned -- exactly the interpolation factor of cross.py:202-204.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "cross.cuh"

namespace qtt {
namespace {

constexpr int NT = 256;

struct ArgMax {
  double v;
  int i;
};

// block-wide (value, index) max, ties to the lower index; every thread gets the result
__device__ ArgMax block_argmax(double v, int i, ArgMax* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) {
      v = v2;
      i = i2;
    }
  }
  __syncthreads();
  if (lane == 0) sh[warp] = {v, i};
  __syncthreads();
  ArgMax best = sh[0];
  for (int w = 1; w < NT / 32; ++w)
    if (sh[w].v > best.v || (sh[w].v == best.v && sh[w].i < best.i)) best = sh[w];
  __syncthreads();
  return best;
}

// Ginv = A[rows]^-1 (r x r) by Gauss-Jordan with partial pivoting on G = [M | I] (r x 2r).
// Returns false when a pivot column is exactly zero (LAPACK getrf's singular case).
__device__ bool invert_rows(const double* A, int r, const int* rows, double* G, double* Ginv, ArgMax* sh) {
  const int w = 2 * r;
  for (int e = threadIdx.x; e < r * w; e += NT) {
    const int i = e / w, c = e - i * w;
    G[e] = c < r ? A[(long long)rows[i] * r + c] : (c - r == i ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int c = 0; c < r; ++c) {
    double v = -1.0;
    int idx = r;
    for (int i = c + threadIdx.x; i < r; i += NT) {
      const double a = fabs(G[i * w + c]);
      if (a > v) {
        v = a;
        idx = i;
      }
    }
    const ArgMax p = block_argmax(v, idx, sh);
    if (!(p.v > 0.0)) return false;
    if (p.i != c)
      for (int k = threadIdx.x; k < w; k += NT) {
        const double t = G[c * w + k];
        G[c * w + k] = G[p.i * w + k];
        G[p.i * w + k] = t;
      }
    __syncthreads();
    const double inv = 1.0 / G[c * w + c];
    __syncthreads();
    for (int k = threadIdx.x; k < w; k += NT) G[c * w + k] *= inv;
    __syncthreads();
    for (int e = threadIdx.x; e < r * w; e += NT) {
      const int i = e / w, k = e - i * w;
      if (i != c && k != c) G[e] -= G[i * w + c] * G[c * w + k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < r; i += NT)
      if (i != c) G[i * w + c] = 0.0;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < r * r; e += NT) Ginv[e] = G[(e / r) * w + r + e % r];
  __syncthreads();
  return true;
}

// B = A Ginv (N x r)
__device__ void apply_inverse(const double* A, int N, int r, const double* Ginv, double* B) {
  for (long long e = threadIdx.x; e < (long long)N * r; e += NT) {
    const long long i = e / r;
    const int j = (int)(e - i * r);
    double s = 0.0;
    for (int k = 0; k < r; ++k) s += A[i * r + k] * Ginv[k * r + j];
    B[e] = s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NT) maxvol_kernel(const double* A, int N, int r, double tol, int max_iters,
                                                     double* W, double* B, double* G, double* Ginv, int* rows,
                                                     int* status) {
  __shared__ ArgMax sh[NT / 32];
  __shared__ double diag0, diagk;
  // ---- 1. pivoted rows (column-pivoted QR of A^T)
  for (long long e = threadIdx.x; e < (long long)N * r; e += NT) W[e] = A[e];
  int* chosen = reinterpret_cast<int*>(Ginv);  // scratch until step 2
  for (int i = threadIdx.x; i < N; i += NT) chosen[i] = 0;
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    double v = -1.0;
    int idx = N;
    for (int i = threadIdx.x; i < N; i += NT) {
      if (chosen[i]) continue;
      double s = 0.0;
      for (int c = 0; c < r; ++c) s += W[(long long)i * r + c] * W[(long long)i * r + c];
      if (s > v) {
        v = s;
        idx = i;
      }
    }
    const ArgMax p = block_argmax(v, idx, sh);
    const double d = sqrt(fmax(p.v, 0.0));
    if (threadIdx.x == 0) {
      rows[k] = p.i;
      chosen[p.i] = 1;
      if (k == 0) diag0 = d;
      diagk = d;
    }
    __syncthreads();
    if (d > 0.0) {  // W_i -= (W_i . u) u, u = W_piv / d
      const double* u = W + (long long)p.i * r;
      for (int i = threadIdx.x; i < N; i += NT) {
        if (i == p.i) continue;
        double s = 0.0;
        for (int c = 0; c < r; ++c) s += W[(long long)i * r + c] * u[c];
        s /= d * d;
        for (int c = 0; c < r; ++c) W[(long long)i * r + c] -= s * u[c];
      }
    }
    __syncthreads();
  }
  const bool deficient = diagk <= 1e-12 * diag0;
  // ---- 2. maxvol swaps
  int st = 0;
  if (deficient) {
    st = 1;
  } else {
    int it = 0;
    for (; it < max_iters; ++it) {
      if (!invert_rows(A, r, rows, G, Ginv, sh)) {
        st = 2;
        break;
      }
      apply_inverse(A, N, r, Ginv, B);
      double v = -1.0;
      int idx = N * r;
      for (long long e = threadIdx.x; e < (long long)N * r; e += NT) {
        const double a = fabs(B[e]);
        if (a > v) {
          v = a;
          idx = (int)e;
        }
      }
      const ArgMax p = block_argmax(v, idx, sh);
      if (p.v <= 1.0 + tol) break;
      if (threadIdx.x == 0) rows[p.i % r] = p.i / r;
      __syncthreads();
    }
    if (st == 0 && it == max_iters) st = 3;
  }
  // ---- B for the returned rows (already current after a tolerance exit); block-collective
  if (st != 0) {
    const bool ok = invert_rows(A, r, rows, G, Ginv, sh);
    if (ok) apply_inverse(A, N, r, Ginv, B);
    if (threadIdx.x == 0 && !ok) st |= 4;
  }
  if (threadIdx.x == 0) *status = st;
}

}  // namespace

int maxvol(Ctx& c, const double* A, int N, int r, double tol, int max_iters, double* B, int* rows_dev,
           int* status_dev) {
  if (N < r || r < 1) throw Error(QTT_ERR_SHAPE, "maxvol needs a tall matrix");
  DBuf W((long long)N * r, c.stream), G(2LL * r * r, c.stream), Ginv((long long)std::max(r * r, N), c.stream);
  maxvol_kernel<<<1, NT, 0, c.stream>>>(A, N, r, tol, max_iters, W.p, B, G.p, Ginv.p, rows_dev, status_dev);
  QTT_CHECK_LAUNCH();
  int st = 0;
  QTT_CUDA(cudaMemcpyAsync(&st, status_dev, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  return st;
}

}  // namespace qtt
