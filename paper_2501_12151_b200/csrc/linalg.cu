// Dense FP64 kernels of the sweep (see linalg.cuh).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "gemm.cuh"
#include "linalg.cuh"
#include "svd_block.cuh"
#include "tma_tile.cuh"

namespace cg = cooperative_groups;

namespace qtt {
namespace {

constexpr int kSmemDoubles = 27 * 1024;  // working sets up to 216 KB stay in shared memory

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum, result broadcast to every thread.  red must hold >= 33 doubles.
template <int NT>
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < NT / 32 ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// ------------------------------------------------------------------ Householder QR
// One CTA.  W is the column-major m x n working copy (shared memory when it fits,
// else global scratch).  tau has k entries.
// (SMEM is a template parameter so the compiler knows W is shared: a runtime choice
// between sm and gws makes W a generic pointer and every access a generic LD/ST)
template <int NT, bool SMEM>
__global__ void __launch_bounds__(NT) qr_kernel(CMatView in, MatView Qo, MatView Ro, double* gws) {
  extern __shared__ double sm[];
  __shared__ double red[40];
  const int m = in.rows, n = in.cols, k = min(m, n);
  double* W = SMEM ? sm : gws;
  double* tau = W + (long long)m * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;

  for (long long e = tid; e < (long long)m * n; e += NT) {
    const int i = (int)(e % m), j = (int)(e / m);
    W[e] = in.p[i * in.rs + j * in.cs];
  }
  __syncthreads();

  for (int j = 0; j < k; ++j) {
    double* vj = W + (long long)j * m;
    double part = 0.0;
    for (int i = j + 1 + tid; i < m; i += NT) part += vj[i] * vj[i];
    const double xnorm2 = block_sum<NT>(part, red);
    const double alpha = vj[j];
    double t = 0.0, beta = alpha, scal = 1.0;
    if (xnorm2 > 0.0) {  // dlarfg
      beta = -copysign(hypot(alpha, sqrt(xnorm2)), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    __syncthreads();
    if (xnorm2 > 0.0)
      for (int i = j + 1 + tid; i < m; i += NT) vj[i] *= scal;
    if (tid == 0) {
      tau[j] = t;
      vj[j] = beta;
    }
    __syncthreads();
    if (t != 0.0) {
      for (int c = j + 1 + warp; c < n; c += NW) {
        double* wc = W + (long long)c * m;
        double w = lane == 0 ? wc[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) w += vj[i] * wc[i];
        w = warp_sum(w) * t;
        if (lane == 0) wc[j] -= w;
        for (int i = j + 1 + lane; i < m; i += 32) wc[i] -= w * vj[i];
      }
    }
    __syncthreads();
  }

  if (Ro.p) {
    for (long long e = tid; e < (long long)k * n; e += NT) {
      const int i = (int)(e % k), c = (int)(e / k);
      Ro.p[i * Ro.rs + c * Ro.cs] = (i <= c) ? W[(long long)c * m + i] : 0.0;
    }
  }
  if (!Qo.p) return;
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {  // dorg2r, in place on columns 0..k-1
    double* vj = W + (long long)j * m;
    const double t = tau[j];
    if (j < k - 1 && t != 0.0) {
      for (int c = j + 1 + warp; c < k; c += NW) {
        double* wc = W + (long long)c * m;
        double w = lane == 0 ? wc[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) w += vj[i] * wc[i];
        w = warp_sum(w) * t;
        if (lane == 0) wc[j] -= w;
        for (int i = j + 1 + lane; i < m; i += 32) wc[i] -= w * vj[i];
      }
    }
    __syncthreads();
    for (int i = tid; i < m; i += NT) {
      if (i > j) vj[i] *= -t;
      else if (i == j) vj[i] = 1.0 - t;
      else vj[i] = 0.0;
    }
    __syncthreads();
  }
  for (long long e = tid; e < (long long)m * k; e += NT) {
    const int i = (int)(e % m), c = (int)(e / m);
    Qo.p[i * Qo.rs + c * Qo.cs] = W[e];
  }
}

// ------------------------------------------------------------------ one-sided Jacobi
// Orthogonalizes the columns of the column-major m x n matrix W (round-robin
// parallel ordering), accumulating V (n x n).  GS lanes own one column pair: each
// lane holds its KMAX-row slice of both columns in registers for the whole rotation
// (one shared-memory read and write per element per round), and the rotation test
// gamma^2 > tol^2 alpha beta needs no square roots.
// Outputs (sorted by descending norm): U = W/sigma (m x n view), s, Vt (n x n view).
template <int GS, int KMAX>
__device__ __forceinline__ bool rotate_pair(double* wa, double* wb, int len, int gl, bool live, double tol2,
                                            double& cs, double& sn) {
  double x[KMAX], y[KMAX];
  double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const int i = gl + k * GS;
    const bool ok = live && i < len;
    x[k] = ok ? wa[i] : 0.0;
    y[k] = ok ? wb[i] : 0.0;
    al = fma(x[k], x[k], al);
    be = fma(y[k], y[k], be);
    ga = fma(x[k], y[k], ga);
  }
#pragma unroll
  for (int o = GS / 2; o > 0; o >>= 1) {
    al += __shfl_xor_sync(0xffffffffu, al, o);
    be += __shfl_xor_sync(0xffffffffu, be, o);
    ga += __shfl_xor_sync(0xffffffffu, ga, o);
  }
  if (!live || ga == 0.0 || !(ga * ga > tol2 * al * be)) return false;
  const double zeta = (be - al) / (2.0 * ga);
  const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
  cs = 1.0 / sqrt(1.0 + t * t);
  sn = cs * t;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const int i = gl + k * GS;
    if (i < len) {
      wa[i] = cs * x[k] - sn * y[k];
      wb[i] = sn * x[k] + cs * y[k];
    }
  }
  return true;
}

template <int GS, int KMAX>
__device__ __forceinline__ void rotate_v(double* va, double* vb, int len, int gl, double cs, double sn) {
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const int i = gl + k * GS;
    if (i < len) {
      const double x = va[i], y = vb[i];
      va[i] = cs * x - sn * y;
      vb[i] = sn * x + cs * y;
    }
  }
}

template <int NT, int GS, int KMAX, bool SMEM>
__global__ void __launch_bounds__(NT) jacobi_kernel(CMatView in, MatView Uo, double* so, MatView Vto,
                                                    double* gws, double tol, int dbg) {
  extern __shared__ double sm[];
  __shared__ int s_rot[2];  // per sweep parity: the reset of sweep s+1 cannot race the reads of sweep s
  int sweeps_done = 0;
  const int m = in.rows, n = in.cols;
  double* W = SMEM ? sm : gws;                          // m x n, column-major
  double* V = W + (long long)m * n;                     // n x n, column-major
  double* sig = V + (long long)n * n;                   // n
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int gl = tid % GS, grp = tid / GS;
  const double tol2 = tol * tol;

  for (long long e = tid; e < (long long)m * n; e += NT) {
    const int i = (int)(e % m), j = (int)(e / m);
    W[e] = in.p[i * in.rs + j * in.cs];
  }
  for (long long e = tid; e < (long long)n * n; e += NT) V[e] = (e % n == e / n) ? 1.0 : 0.0;
  __syncthreads();

  const int P = n + (n & 1);  // players incl. a dummy when n is odd
  for (int sweep = 0; sweep < 80; ++sweep) {
    if (tid == 0) s_rot[sweep & 1] = 0;
    __syncthreads();
    int rotated = 0;
    for (int r = 0; r < P - 1; ++r) {
      // every thread runs the same passes (the group shuffles need whole warps)
      for (int base = 0; base < P / 2; base += NT / GS) {
        const int q = base + grp;
        int a = 0, b = 0;
        if (q == 0) { a = r; b = P - 1; }
        else { a = (r + q) % (P - 1); b = (r - q + (P - 1)) % (P - 1); }
        const bool live = q < P / 2 && a < n && b < n;
        if (a > b) { const int t = a; a = b; b = t; }
        if (!live) { a = 0; b = 0; }
        double cs = 1.0, sn = 0.0;
        if (rotate_pair<GS, KMAX>(W + (long long)a * m, W + (long long)b * m, m, gl, live, tol2, cs, sn)) {
          rotate_v<GS, KMAX>(V + (long long)a * n, V + (long long)b * n, n, gl, cs, sn);
          rotated = 1;
        }
      }
      __syncthreads();
    }
    if (rotated) s_rot[sweep & 1] = 1;
    __syncthreads();
    sweeps_done = sweep + 1;
    if (!s_rot[sweep & 1]) break;
  }
  if (dbg && tid == 0) printf("[qtt] jacobi %dx%d sweeps %d\n", m, n, sweeps_done);
  // column norms
  for (int c = warp; c < n; c += NW) {
    const double* wc = W + (long long)c * m;
    double s2 = 0;
    for (int i = lane; i < m; i += 32) s2 += wc[i] * wc[i];
    s2 = warp_sum(s2);
    if (lane == 0) sig[c] = sqrt(s2);
  }
  __syncthreads();
  // stable descending rank of each column, then scatter
  for (int c = tid; c < n; c += NT) {
    const double sc = sig[c];
    int rank = 0;
    for (int d = 0; d < n; ++d) {
      const double sd = sig[d];
      rank += (sd > sc) || (sd == sc && d < c);
    }
    so[rank] = sc;
    // U column rank = w_c / sigma_c  (unit basis vector when sigma_c == 0)
    const double inv = sc > 0 ? 1.0 / sc : 0.0;
    const double* wc = W + (long long)c * m;
    if (Uo.p)
      for (int i = 0; i < m; ++i)
        Uo.p[i * Uo.rs + rank * Uo.cs] = sc > 0 ? wc[i] * inv : (i == rank ? 1.0 : 0.0);
    if (Vto.p) {
      const double* vc = V + (long long)c * n;
      for (int i = 0; i < n; ++i) Vto.p[rank * Vto.rs + i * Vto.cs] = vc[i];
    }
  }
}

// One-sided Jacobi for the square case (the R^T of svd_tall): W (n x n) and V (n x n)
// stacked into one column-major array, each padded to SEG = 16 K rows with zeros (zero
// rows stay zero under rotations), column stride 2 SEG.  GS = 8 lanes own a column pair
// and move 16-byte (double2) chunks: one group covers 16 rows per chunk, so every
// quarter-warp access is one contiguous 128-byte line (no bank conflicts) and the
// shared-memory instruction count is half that of scalar access.  W and V chunks are
// loaded together (V's loads no longer wait for the rotation angle), warps whose pairs
// are all past P/2 skip the round, and the three dot products run in two chains each.
// (tools/svd_bench.py; ncu of the scalar kernel: issue-bound, fp64 pipe 27% active.)
__device__ __forceinline__ bool jac_angle(double al, double be, double ga, double tol2, double& cs, double& sn) {
  if (ga == 0.0 || !(ga * ga > tol2 * al * be)) return false;
  const double zeta = (be - al) / (2.0 * ga);
  const double az = fabs(zeta);
  // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)); for huge |zeta|, t = 1 / (2 zeta)
  const double t = az < 1e100 ? copysign(1.0 / (az + sqrt(fma(az, az, 1.0))), zeta) : 0.5 / zeta;
  cs = 1.0 / sqrt(fma(t, t, 1.0));
  sn = cs * t;
  return true;
}

template <int NT, int K, bool VLATE = (K >= 7)>
__global__ void __launch_bounds__(NT) jacobi_sq_kernel(CMatView in, MatView Uo, double* so, MatView Vto, double tol,
                                                       int dbg) {
  constexpr int GS = 8, SEG = 16 * K, LD = 2 * SEG;
  extern __shared__ double sm[];
  __shared__ int s_rot[2];  // per sweep parity: the reset of sweep s+1 cannot race the reads of sweep s
  const int n = in.cols;
  double* S = sm;  // n columns of LD doubles
  double* sig = S + (long long)LD * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int gl = tid % GS, grp = tid / GS;
  const double tol2 = tol * tol;
  for (int e = tid; e < LD * n; e += NT) {
    const int i = e % LD, j = e / LD;
    double v = 0.0;
    if (i < n) v = in.p[i * in.rs + j * in.cs];
    else if (i >= SEG && i - SEG == j) v = 1.0;
    S[e] = v;
  }
  __syncthreads();
  int sweeps_done = 0;
  const int P = n + (n & 1), half = P / 2;
  const bool warp_live = warp * (32 / GS) < half;
  for (int sweep = 0; sweep < 80; ++sweep) {
    if (tid == 0) s_rot[sweep & 1] = 0;
    __syncthreads();
    int rotated = 0;
    for (int r = 0; r < P - 1; ++r) {
      if (warp_live) {
        const int q = grp;
        int a, b;
        if (q == 0) { a = r; b = P - 1; }
        else { a = (r + q) % (P - 1); b = (r - q + (P - 1)) % (P - 1); }
        const bool live = q < half && a < n && b < n;
        if (a > b) { const int t = a; a = b; b = t; }
        if (!live) { a = 0; b = 0; }
        double2* wa = reinterpret_cast<double2*>(S + (long long)a * LD) + gl;
        double2* wb = reinterpret_cast<double2*>(S + (long long)b * LD) + gl;
        // chunks 0..K-1: W rows, K..2K-1: V rows (V loaded after the angle when K = 7: the
        // 448-thread block is capped at 128 registers)
        constexpr int KR = VLATE ? K : 2 * K;
        double2 x[KR], y[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          x[k] = wa[k * GS];
          y[k] = wb[k * GS];
        }
        double al0 = 0.0, be0 = 0.0, ga0 = 0.0, al1 = 0.0, be1 = 0.0, ga1 = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          al0 = fma(x[k].x, x[k].x, al0); be0 = fma(y[k].x, y[k].x, be0); ga0 = fma(x[k].x, y[k].x, ga0);
          al1 = fma(x[k].y, x[k].y, al1); be1 = fma(y[k].y, y[k].y, be1); ga1 = fma(x[k].y, y[k].y, ga1);
        }
        double al = al0 + al1, be = be0 + be1, ga = ga0 + ga1;
#pragma unroll
        for (int o = GS / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        double cs, sn;
        if (live && jac_angle(al, be, ga, tol2, cs, sn)) {
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            wa[k * GS] = make_double2(cs * x[k].x - sn * y[k].x, cs * x[k].y - sn * y[k].y);
            wb[k * GS] = make_double2(sn * x[k].x + cs * y[k].x, sn * x[k].y + cs * y[k].y);
          }
          if constexpr (VLATE) {
#pragma unroll
            for (int k = K; k < 2 * K; ++k) {
              const double2 u = wa[k * GS], v = wb[k * GS];
              wa[k * GS] = make_double2(cs * u.x - sn * v.x, cs * u.y - sn * v.y);
              wb[k * GS] = make_double2(sn * u.x + cs * v.x, sn * u.y + cs * v.y);
            }
          }
          rotated = 1;
        }
      }
      __syncthreads();
    }
    if (rotated) s_rot[sweep & 1] = 1;
    __syncthreads();
    sweeps_done = sweep + 1;
    if (!s_rot[sweep & 1]) break;
  }
  if (dbg && tid == 0) printf("[qtt] jacobi(sq) %dx%d sweeps %d\n", n, n, sweeps_done);
  for (int c = warp; c < n; c += NW) {
    const double* wc = S + (long long)c * LD;
    double s2 = 0;
    for (int i = lane; i < n; i += 32) s2 += wc[i] * wc[i];
    s2 = warp_sum(s2);
    if (lane == 0) sig[c] = sqrt(s2);
  }
  __syncthreads();
  for (int c = tid; c < n; c += NT) {
    const double sc = sig[c];
    int rank = 0;
    for (int d = 0; d < n; ++d) {
      const double sd = sig[d];
      rank += (sd > sc) || (sd == sc && d < c);
    }
    so[rank] = sc;
    const double inv = sc > 0 ? 1.0 / sc : 0.0;
    const double* wc = S + (long long)c * LD;
    if (Uo.p)
      for (int i = 0; i < n; ++i)
        Uo.p[i * Uo.rs + rank * Uo.cs] = sc > 0 ? wc[i] * inv : (i == rank ? 1.0 : 0.0);
    if (Vto.p)
      for (int i = 0; i < n; ++i) Vto.p[rank * Vto.rs + i * Vto.cs] = wc[SEG + i];
  }
}

// ------------------------------------------------------------------ Cholesky
constexpr int CB = 64;  // Cholesky block size

// Factor the diagonal block A[j0:j0+nb, j0:j0+nb] in shared memory.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double* A, int dim, long long ld, int j0,
                                                         int* info) {
  if (*info != 0) return;
  __shared__ double a[CB][CB + 1];
  __shared__ int bad;
  const int nb = min(CB, dim - j0);
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += 256) {
    const int i = e / nb, j = e % nb;
    a[i][j] = A[(j0 + i) * ld + j0 + j];
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double d = a[j][j];
    if (!(d > 0.0)) {  // dpotrf: non-positive or NaN pivot
      if (tid == 0) { bad = 1; atomicCAS(info, 0, j0 + j + 1); }
      __syncthreads();
      break;
    }
    const double ljj = sqrt(d);
    __syncthreads();
    if (tid == 0) a[j][j] = ljj;
    for (int i = j + 1 + tid; i < nb; i += 256) a[i][j] /= ljj;
    __syncthreads();
    // trailing update of the block's lower triangle
    const int rem = nb - j - 1;
    for (int e = tid; e < rem * rem; e += 256) {
      const int i = j + 1 + e / rem, c = j + 1 + e % rem;
      if (c <= i) a[i][c] -= a[i][j] * a[c][j];
    }
    __syncthreads();
  }
  if (bad) return;
  for (int e = tid; e < nb * nb; e += 256) {
    const int i = e / nb, j = e % nb;
    if (j <= i) A[(j0 + i) * ld + j0 + j] = a[i][j];
  }
}

// Panel solve L21 = A21 L11^{-T} for rows j0+nb .. dim-1 (one thread per row).
__global__ void __launch_bounds__(128) potrf_trsm_kernel(double* A, int dim, long long ld, int j0,
                                                         const int* info) {
  if (*info != 0) return;
  __shared__ double L[CB][CB + 1];
  const int nb = min(CB, dim - j0);
  for (int e = threadIdx.x; e < nb * nb; e += 128) {
    const int i = e / nb, j = e % nb;
    L[i][j] = (j <= i) ? A[(j0 + i) * ld + j0 + j] : 0.0;
  }
  __syncthreads();
  const int row = j0 + nb + blockIdx.x * 128 + threadIdx.x;
  if (row >= dim) return;
  double x[CB];
  double* a = A + row * ld + j0;
#pragma unroll
  for (int j = 0; j < CB; ++j) x[j] = j < nb ? a[j] : 0.0;
#pragma unroll
  for (int j = 0; j < CB; ++j) {
    if (j < nb) {
      double v = x[j];
#pragma unroll
      for (int p = 0; p < j; ++p) v -= x[p] * L[j][p];
      x[j] = v / L[j][j];
    }
  }
#pragma unroll
  for (int j = 0; j < CB; ++j)
    if (j < nb) a[j] = x[j];
}

// Forward then backward substitution with L (lower, row-major) in one CTA, blocked
// by 32 rows: each block's 32x32 triangle is solved by one warp, the remaining
// right-hand side is updated by all warps (GEMV on the panel below/above).
__global__ void __launch_bounds__(1024) potrs_kernel(const double* L, int dim, long long ld, double* b) {
  __shared__ double xb[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // forward: L y = b
  for (int j0 = 0; j0 < dim; j0 += 32) {
    const int nb = min(32, dim - j0);
    if (warp == 0) {
      double v = lane < nb ? b[j0 + lane] : 0.0;
      for (int j = 0; j < nb; ++j) {
        const double lij = lane < nb ? L[(j0 + lane) * ld + j0 + j] : 0.0;
        const double xj = __shfl_sync(0xffffffffu, v, j) / L[(j0 + j) * ld + j0 + j];
        if (lane == j) v = xj;
        else if (lane > j) v -= lij * xj;
      }
      if (lane < nb) { b[j0 + lane] = v; xb[lane] = v; }
    }
    __syncthreads();
    for (int i = j0 + nb + tid; i < dim; i += 1024) {
      double s = 0.0;
      const double* li = L + i * ld + j0;
      for (int j = 0; j < nb; ++j) s += li[j] * xb[j];
      b[i] -= s;
    }
    __syncthreads();
  }
  // backward: L^T x = y
  for (int j1 = dim; j1 > 0; j1 -= 32) {
    const int j0 = max(0, j1 - 32), nb = j1 - j0;
    if (warp == 0) {
      double v = lane < nb ? b[j0 + lane] : 0.0;
      for (int j = nb - 1; j >= 0; --j) {
        // L^T[lane, j] = L[j0+j, j0+lane]
        const double lji = lane < nb ? L[(j0 + j) * ld + j0 + lane] : 0.0;
        const double xj = __shfl_sync(0xffffffffu, v, j) / L[(j0 + j) * ld + j0 + j];
        if (lane == j) v = xj;
        else if (lane < j) v -= lji * xj;
      }
      if (lane < nb) { b[j0 + lane] = v; xb[lane] = v; }
    }
    __syncthreads();
    // b[i] -= sum_j L[j0+j, i] x[j]  for i < j0  (column access: rows j0..j1 of L, coalesced in i)
    for (int i = tid; i < j0; i += 1024) {
      double s = 0.0;
      for (int j = 0; j < nb; ++j) s += L[(j0 + j) * ld + i] * xb[j];
      b[i] -= s;
    }
    __syncthreads();
  }
}

__global__ void row_abs_sum_kernel(const double* A, int dim, long long ld, double* out) {
  // one warp per row; max over rows via integer atomicMax on non-negative doubles
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= dim) return;
  const double* a = A + row * ld;
  double s = 0.0;
  for (int j = lane; j < dim; j += 32) s += fabs(a[j]);
  s = warp_sum(s);
  if (lane == 0) atomicMax((unsigned long long*)out, (unsigned long long)__double_as_longlong(s));
}

// ------------------------------------------------------------------ reductions
constexpr int RED_BLOCKS = 296;

template <int MODE>  // 0: dot(a,b)  1: sum(a)  2: sqrt(dot(a,a))
__global__ void __launch_bounds__(256) reduce_kernel(const double* a, const double* b, long long n,
                                                     double* partial, unsigned* counter, double* out) {
  __shared__ double red[40];
  __shared__ bool last;
  double s = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    if (MODE == 0) s += a[i] * b[i];
    else if (MODE == 1) s += a[i];
    else s += a[i] * a[i];
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = s;
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += 256) v += ((volatile double*)partial)[i];
  v = block_sum<256>(v, red);
  if (threadIdx.x == 0) {
    *out = MODE == 2 ? sqrt(v) : v;
    *counter = 0u;
  }
}

template <int MODE>
void reduce(Ctx& c, const double* a, const double* b, long long n, double* out) {
  const int blocks = (int)std::max<long long>(1, std::min<long long>(RED_BLOCKS, cdiv(n, 256)));
  reduce_kernel<MODE><<<blocks, 256, 0, c.stream>>>(a, b, n, c.red_partial, c.red_counter, out);
  QTT_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ elementwise
// One CTA per output row (a, xx, mm): y[row, (b, yy)] = sum_n A[a,mm,n,b] x[xx,n,yy].  The
// row's operator column A[a,mm,:,:] and vector slice x[xx,:,:] are staged in shared memory,
// the row (Ra1 * rx1 doubles, contiguous) is written with coalesced streaming stores --
// the kernel is a pure HBM write stream (tt.py:443-447).
__global__ void __launch_bounds__(256) kron_core_kernel(const double* __restrict__ A, int Ra0, int m, int n,
                                                        int Ra1, const double* __restrict__ x, int rx0, int rx1,
                                                        double* __restrict__ y, int staged) {
  extern __shared__ double sh[];
  const long long rows = (long long)Ra0 * rx0 * m;
  const int cols = Ra1 * rx1;
  for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
    const int mm = (int)(row % m);
    const long long t = row / m;
    const int xx = (int)(t % rx0), a = (int)(t / rx0);
    const double* sa = A + ((long long)a * m + mm) * n * Ra1;  // A[a,mm,nn,b] at nn*Ra1 + b
    const double* sx = x + (long long)xx * n * rx1;            // x[xx,nn,yy] at nn*rx1 + yy
    if (staged) {  // (else: read through L1/L2 -- only for ranks beyond the shared-memory stage)
      __syncthreads();
      for (int i = threadIdx.x; i < n * Ra1; i += blockDim.x) sh[i] = sa[i];
      for (int i = threadIdx.x; i < n * rx1; i += blockDim.x) sh[n * Ra1 + i] = sx[i];
      __syncthreads();
      sa = sh;
      sx = sh + n * Ra1;
    }
    double* yr = y + row * cols;
    if ((rx1 & 1) == 0 && (cols & 1) == 0) {  // pairs of yy: 16-byte streaming stores, no division
      const int h = rx1 >> 1;  // (b, j) pairs flattened: every thread busy even when rx1 < 2 * blockDim
      double2* dst = reinterpret_cast<double2*>(yr);
      for (int e = threadIdx.x; e < Ra1 * h; e += blockDim.x) {
        const int b = e / h, j = e - b * h;
        double s0 = 0.0, s1 = 0.0;
        for (int nn = 0; nn < n; ++nn) {
          const double av = sa[nn * Ra1 + b];
          s0 = fma(av, sx[nn * rx1 + 2 * j], s0);
          s1 = fma(av, sx[nn * rx1 + 2 * j + 1], s1);
        }
        __stcs(dst + e, make_double2(s0, s1));
      }
    } else {
      for (int e = threadIdx.x; e < cols; e += blockDim.x) {
        const int b = e / rx1, yy = e - b * rx1;
        double s = 0.0;
        for (int nn = 0; nn < n; ++nn) s += sa[nn * Ra1 + b] * sx[nn * rx1 + yy];
        __stcs(yr + e, s);
      }
    }
  }
}

__global__ void scale_rows_kernel(const double* in, long long ld_in, const double* scale, int rows,
                                  int cols, double* out, long long ld_out) {
  const long long total = (long long)rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols), j = (int)(e % cols);
    out[i * ld_out + j] = scale[i] * in[i * ld_in + j];
  }
}

__global__ void copy_view_kernel(CMatView in, MatView out) {
  const long long total = (long long)in.rows * in.cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / in.cols), j = (int)(e % in.cols);
    out.p[i * out.rs + j * out.cs] = in.p[i * in.rs + j * in.cs];
  }
}

__global__ void fill_kernel(double* p, long long n, double v) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    p[e] = v;
}

__global__ void axpby_kernel(long long n, double a, const double* x, double b, double* y) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    y[e] = a * x[e] + b * y[e];
}

__global__ void op_core_diag_kernel(const double* A, int R0, int m, int R1, double* d) {
  const long long total = (long long)R0 * m * R1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(e % R1), mm = (int)((e / R1) % m), a = (int)(e / ((long long)R1 * m));
    d[e] = A[(((long long)a * m + mm) * m + mm) * R1 + b];
  }
}

inline int grid_for(long long n) { return (int)std::max<long long>(1, std::min<long long>(cdiv(n, 256), 1184)); }

}  // namespace

// ------------------------------------------------------------------ host wrappers
void qr(Ctx& c, CMatView in, MatView Q, MatView R) {
  const int m = in.rows, n = in.cols;
  if (m <= 0 || n <= 0) return;
  const int k = std::min(m, n);
  const long long need = (long long)m * n + k;
  constexpr int NT = 512;
  c.stats.qr_calls++;
  if (need > kSmemDoubles && k >= 64) {  // past one CTA's shared memory: blocked multi-CTA QR
    qr_large(c, in, Q, R);
    return;
  }
  static const bool cta = !(std::getenv("QTT_QR_CTA") && std::atoi(std::getenv("QTT_QR_CTA")) == 0);
  if (cta && n <= 256 && m <= 1024 && qr_cta_smem_doubles(m, n) * 8 <= 224 * 1024) {
    qr_cta(c, in, Q, R);
    return;
  }
  if (need <= kSmemDoubles) {
    static PerDevice<bool> attr_dev(false);
    bool& attr = attr_dev();
    if (!attr) {
      QTT_CUDA(cudaFuncSetAttribute(qr_kernel<NT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmemDoubles * 8));
      attr = true;
    }
    qr_kernel<NT, true><<<1, NT, need * 8, c.stream>>>(in, Q, R, nullptr);
    QTT_CHECK_LAUNCH();
  } else {
    DBuf ws(need, c.stream);
    qr_kernel<NT, false><<<1, NT, 0, c.stream>>>(in, Q, R, ws.p);
    QTT_CHECK_LAUNCH();
  }
}

static int jacobi_dbg() {
  static const int on = std::getenv("QTT_DEBUG_JACOBI") != nullptr;
  return on;
}

template <int GS, int KMAX>
static void jacobi_launch(Ctx& c, CMatView in, MatView U, double* s, MatView Vt, double tol) {
  // few lanes per pair and few warps: the rotation arithmetic is issued once per warp,
  // so a round costs ~(warps x instructions) -- 256 threads cover 64 pairs at GS = 4
  constexpr int NT = 256;
  const int m = in.rows, n = in.cols;
  const long long need = (long long)m * n + (long long)n * n + n;
  if (need <= kSmemDoubles) {
    auto kern = jacobi_kernel<NT, GS, KMAX, true>;
    static PerDevice<bool> attr_dev(false);
    bool& attr = attr_dev();
    if (!attr) {
      QTT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDoubles * 8));
      attr = true;
    }
    kern<<<1, NT, need * 8, c.stream>>>(in, U, s, Vt, nullptr, tol, jacobi_dbg());
    QTT_CHECK_LAUNCH();
  } else {
    DBuf ws(need, c.stream);
    jacobi_kernel<NT, GS, KMAX, false><<<1, NT, 0, c.stream>>>(in, U, s, Vt, ws.p, tol, jacobi_dbg());
    QTT_CHECK_LAUNCH();
  }
}

// ---- the same square one-sided Jacobi on a 2-CTA cluster: CTA 0 holds W, finds the angles and
// rotates W; CTA 1 holds V and applies the same rotations one hop behind.  The dependency is
// one-way (V never feeds an angle), so the DSMEM hop is a pipeline delay, not a per-round round
// trip (the row-split cluster variants measured earlier paid one per round).  Each CTA moves half
// of the shared-memory traffic that bounds the single-CTA kernel.  Per round CTA 0's group
// leaders store (cs, sn) into a ring slot of CTA 1's shared memory, thread 0 then arrives
// (release.cluster) on that slot's mbarrier in CTA 1; CTA 1 hands the slot back through an
// mbarrier in CTA 0.  After the last sweep CTA 0 sends the column ranks with a STOP header.
// Every floating-point operation and its order are those of jacobi_sq_kernel: same bits.
namespace jq2 {
constexpr int DEPTH = 8;     // ring slots
constexpr int MAXG = 80;     // rotation groups per round (<= 8 K = 80)
struct Mail {                // lives in CTA 1's shared memory (CTA 0 writes it remotely)
  double cs[DEPTH][MAXG];
  double sn[DEPTH][MAXG];
  int hdr[DEPTH];            // 0: a round's rotations, 1: stop (rank[] is valid)
  int rank[128];
};
__device__ __forceinline__ unsigned map_remote(const void* p, unsigned cta) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
__device__ __forceinline__ void remote_arrive(unsigned remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void st_remote_f64(unsigned addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_remote_s32(unsigned addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
}  // namespace jq2

template <int NT, int K>
__global__ void __launch_bounds__(NT) jacobi_sq2_kernel(CMatView in, MatView Uo, double* so, MatView Vto,
                                                        double tol, int dbg) {
  constexpr int GS = 8, SEG = 16 * K;
  extern __shared__ double sm[];
  __shared__ int s_rot[2];
  __shared__ jq2::Mail mail;                       // used in CTA 1
  __shared__ __align__(8) uint64_t full[jq2::DEPTH];   // used in CTA 1: slot filled by CTA 0
  __shared__ __align__(8) uint64_t empty[jq2::DEPTH];  // used in CTA 0: slot released by CTA 1
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank_in_cl = cl.block_rank();
  const int n = in.cols;
  double* S = sm;  // n columns of SEG doubles: W in CTA 0, V in CTA 1
  double* sig = S + (long long)SEG * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  const int gl = tid % GS, grp = tid / GS;
  const double tol2 = tol * tol;
  if (tid == 0) {
    for (int i = 0; i < jq2::DEPTH; ++i) {
      tma::mbar_init(&full[i], 1);
      tma::mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int e = tid; e < SEG * n; e += NT) {
    const int i = e % SEG, j = e / SEG;
    double v = 0.0;
    if (rank_in_cl == 0) {
      if (i < n) v = in.p[i * in.rs + j * in.cs];
    } else if (i == j) {
      v = 1.0;
    }
    S[e] = v;
  }
  cl.sync();
  const int P = n + (n & 1), half = P / 2;
  const bool warp_live = warp * (32 / GS) < half;
  auto pair_of = [&](int r, int& a, int& b) {
    const int q = grp;
    if (q == 0) { a = r; b = P - 1; }
    else { a = (r + q) % (P - 1); b = (r - q + (P - 1)) % (P - 1); }
    const bool live = q < half && a < n && b < n;
    if (a > b) { const int t = a; a = b; b = t; }
    if (!live) { a = 0; b = 0; }
    return live;
  };
  if (rank_in_cl == 0) {
    // ---------------- CTA 0: W, the angles, the convergence decision
    const unsigned r_cs = jq2::map_remote(&mail.cs[0][0], 1), r_sn = jq2::map_remote(&mail.sn[0][0], 1);
    const unsigned r_hdr = jq2::map_remote(&mail.hdr[0], 1), r_rank = jq2::map_remote(&mail.rank[0], 1);
    const unsigned r_full = jq2::map_remote(&full[0], 1);
    unsigned t = 0;  // rounds sent so far
    int sweeps_done = 0;
    for (int sweep = 0; sweep < 80; ++sweep) {
      if (tid == 0) s_rot[sweep & 1] = 0;
      __syncthreads();
      int rotated = 0;
      for (int r = 0; r < P - 1; ++r, ++t) {
        const unsigned slot = t % jq2::DEPTH;
        if (warp_live) {
          int a, b;
          const bool live = pair_of(r, a, b);
          double2* wa = reinterpret_cast<double2*>(S + (long long)a * SEG) + gl;
          double2* wb = reinterpret_cast<double2*>(S + (long long)b * SEG) + gl;
          double2 x[K], y[K];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            x[k] = wa[k * GS];
            y[k] = wb[k * GS];
          }
          double al0 = 0.0, be0 = 0.0, ga0 = 0.0, al1 = 0.0, be1 = 0.0, ga1 = 0.0;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            al0 = fma(x[k].x, x[k].x, al0); be0 = fma(y[k].x, y[k].x, be0); ga0 = fma(x[k].x, y[k].x, ga0);
            al1 = fma(x[k].y, x[k].y, al1); be1 = fma(y[k].y, y[k].y, be1); ga1 = fma(x[k].y, y[k].y, ga1);
          }
          double al = al0 + al1, be = be0 + be1, ga = ga0 + ga1;
#pragma unroll
          for (int o = GS / 2; o > 0; o >>= 1) {
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
            ga += __shfl_xor_sync(0xffffffffu, ga, o);
          }
          double cs = 2.0, sn = 0.0;  // cs = 2: no rotation
          const bool rot = live && jac_angle(al, be, ga, tol2, cs, sn);
          if (!rot) cs = 2.0;
          if (gl == 0) {
            if (t >= (unsigned)jq2::DEPTH) jq2::wait_cluster(&empty[slot], ((t / jq2::DEPTH) - 1) & 1u);
            jq2::st_remote_f64(r_cs + (slot * jq2::MAXG + grp) * 8, cs);
            jq2::st_remote_f64(r_sn + (slot * jq2::MAXG + grp) * 8, sn);
          }
          if (rot) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
              wa[k * GS] = make_double2(cs * x[k].x - sn * y[k].x, cs * x[k].y - sn * y[k].y);
              wb[k * GS] = make_double2(sn * x[k].x + cs * y[k].x, sn * x[k].y + cs * y[k].y);
            }
            rotated = 1;
          }
        }
        if (tid == 0) {
          if (t >= (unsigned)jq2::DEPTH) jq2::wait_cluster(&empty[slot], ((t / jq2::DEPTH) - 1) & 1u);
          jq2::st_remote_s32(r_hdr + slot * 4, 0);
        }
        __syncthreads();
        if (tid == 0) jq2::remote_arrive(r_full + slot * 8);
      }
      if (rotated) s_rot[sweep & 1] = 1;
      __syncthreads();
      sweeps_done = sweep + 1;
      if (!s_rot[sweep & 1]) break;
    }
    if (dbg && tid == 0) printf("[qtt] jacobi(sq2) %dx%d sweeps %d\n", n, n, sweeps_done);
    for (int c = warp; c < n; c += NW) {
      const double* wc = S + (long long)c * SEG;
      double s2 = 0;
      for (int i = lane; i < n; i += 32) s2 += wc[i] * wc[i];
      s2 = warp_sum(s2);
      if (lane == 0) sig[c] = sqrt(s2);
    }
    __syncthreads();
    const unsigned slot = t % jq2::DEPTH;
    if (tid == 0 && t >= (unsigned)jq2::DEPTH) jq2::wait_cluster(&empty[slot], ((t / jq2::DEPTH) - 1) & 1u);
    __syncthreads();
    for (int c = tid; c < n; c += NT) {
      const double sc = sig[c];
      int rank = 0;
      for (int d = 0; d < n; ++d) {
        const double sd = sig[d];
        rank += (sd > sc) || (sd == sc && d < c);
      }
      jq2::st_remote_s32(r_rank + c * 4, rank);
      so[rank] = sc;
      const double inv = sc > 0 ? 1.0 / sc : 0.0;
      const double* wc = S + (long long)c * SEG;
      if (Uo.p)
        for (int i = 0; i < n; ++i)
          Uo.p[i * Uo.rs + rank * Uo.cs] = sc > 0 ? wc[i] * inv : (i == rank ? 1.0 : 0.0);
    }
    if (tid == 0) jq2::st_remote_s32(r_hdr + slot * 4, 1);
    __syncthreads();
    if (tid == 0) jq2::remote_arrive(r_full + slot * 8);
  } else {
    // ---------------- CTA 1: V, one hop behind
    const unsigned r_empty = jq2::map_remote(&empty[0], 0);
    unsigned t = 0;
    for (;; ++t) {
      const unsigned slot = t % jq2::DEPTH;
      jq2::wait_cluster(&full[slot], (t / jq2::DEPTH) & 1u);
      if (mail.hdr[slot] != 0) break;
      const int r = (int)(t % (unsigned)(P - 1));
      if (warp_live) {
        int a, b;
        pair_of(r, a, b);
        const double cs = mail.cs[slot][grp], sn = mail.sn[slot][grp];
        if (cs != 2.0) {
          double2* wa = reinterpret_cast<double2*>(S + (long long)a * SEG) + gl;
          double2* wb = reinterpret_cast<double2*>(S + (long long)b * SEG) + gl;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const double2 u = wa[k * GS], v = wb[k * GS];
            wa[k * GS] = make_double2(cs * u.x - sn * v.x, cs * u.y - sn * v.y);
            wb[k * GS] = make_double2(sn * u.x + cs * v.x, sn * u.y + cs * v.y);
          }
        }
      }
      __syncthreads();
      if (tid == 0) jq2::remote_arrive(r_empty + slot * 8);
    }
    if (Vto.p)
      for (int c = tid; c < n; c += NT) {
        const int rank = mail.rank[c];
        const double* vc = S + (long long)c * SEG;
        for (int i = 0; i < n; ++i) Vto.p[rank * Vto.rs + i * Vto.cs] = vc[i];
      }
  }
  cl.sync();  // neither CTA leaves while the other may still write its shared memory
}

template <int NT, int K>
static bool jacobi_sq2_launch(Ctx& c, CMatView in, MatView U, double* s, MatView Vt, double tol) {
  static PerDevice<int> ok_dev(-1);
  int& ok = ok_dev();
  const size_t bytes = ((size_t)16 * K * in.cols + in.cols) * sizeof(double);
  if (ok < 0) {
    // the widest matrix of this K (n = 16 K) next to ~11 KB of static shared memory (the mail box)
    ok = cudaFuncSetAttribute(jacobi_sq2_kernel<NT, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(((size_t)16 * K * 16 * K + 16 * K) * sizeof(double))) == cudaSuccess ? 1 : 0;
    cudaGetLastError();
  }
  if (!ok) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, jacobi_sq2_kernel<NT, K>, in, U, s, Vt, tol, jacobi_dbg());
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  QTT_CHECK_LAUNCH();
  return true;
}

// n <= 16 K: 8 lanes per pair, ceil(n/2) <= 8 K pairs -> NT = 64 K threads
template <int NT, int K>
static void jacobi_sq_launch(Ctx& c, CMatView in, MatView U, double* s, MatView Vt, double tol, size_t bytes) {
  static_assert(NT == 64 * K, "one 8-lane group per pair");
  static PerDevice<bool> attr_dev(false);
  bool& attr = attr_dev();
  if (!attr) {
    QTT_CUDA(cudaFuncSetAttribute(jacobi_sq_kernel<NT, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemDoubles * 8));
    attr = true;
  }
  jacobi_sq_kernel<NT, K><<<1, NT, bytes, c.stream>>>(in, U, s, Vt, tol, jacobi_dbg());
  QTT_CHECK_LAUNCH();
}

static void jacobi(Ctx& c, CMatView in, MatView U, double* s, MatView Vt) {
  const int m = in.rows, n = in.cols;
  static const int big_at = std::getenv("QTT_BJ_MIN") ? std::atoi(std::getenv("QTT_BJ_MIN")) : 160;
  if (std::min(m, n) >= big_at) {
    svd_block_jacobi(c, in, U, s, Vt);
    return;
  }
  const double tol = std::sqrt((double)m) * 2.220446049250313e-16;
  static const int sq = std::getenv("QTT_JAC_SQ") ? std::atoi(std::getenv("QTT_JAC_SQ")) : 1;
  // (The 2-CTA kernel also fits widths 113..144 -- W alone and V alone fit a CTA's shared memory --
  // and is faster there than the block Jacobi, tools/svd_mid2.py: n = 120 2.22 vs 2.83 ms, 140
  // 2.85 vs 3.45; it loses from 150 on.  Not routed: 0.09 s of C5's 1.8 s SVD phase, and another
  // SVD algorithm at those widths moves C5's trajectory.)
  if (sq && m == n && n <= 112) {
    const int K = cdiv(n, 16);
    const size_t bytes = ((size_t)32 * K * n + n) * sizeof(double);
    // two CTAs (W | V) from n = 81 on (200 x 100: 2.48 -> 2.14 ms); below, a round is latency-
    // rather than shared-memory-bound and the split does not pay (136 x 68: 1.09 -> 1.13 ms).
    // QTT_JAC_SQ2 = smallest K = ceil(n / 16) that takes the cluster kernel (0: never).
    static const int sq2 = std::getenv("QTT_JAC_SQ2") ? std::atoi(std::getenv("QTT_JAC_SQ2")) : 6;
    if (sq2 > 0 && K >= std::max(3, sq2)) {
      bool done = false;
      switch (K) {
        case 3: done = jacobi_sq2_launch<192, 3>(c, in, U, s, Vt, tol); break;
        case 4: done = jacobi_sq2_launch<256, 4>(c, in, U, s, Vt, tol); break;
        case 5: done = jacobi_sq2_launch<320, 5>(c, in, U, s, Vt, tol); break;
        case 6: done = jacobi_sq2_launch<384, 6>(c, in, U, s, Vt, tol); break;
        default: done = jacobi_sq2_launch<448, 7>(c, in, U, s, Vt, tol); break;
      }
      if (done) return;
    }
    switch (K) {
      case 1: jacobi_sq_launch<64, 1>(c, in, U, s, Vt, tol, bytes); break;
      case 2: jacobi_sq_launch<128, 2>(c, in, U, s, Vt, tol, bytes); break;
      case 3: jacobi_sq_launch<192, 3>(c, in, U, s, Vt, tol, bytes); break;
      case 4: jacobi_sq_launch<256, 4>(c, in, U, s, Vt, tol, bytes); break;
      case 5: jacobi_sq_launch<320, 5>(c, in, U, s, Vt, tol, bytes); break;
      case 6: jacobi_sq_launch<384, 6>(c, in, U, s, Vt, tol, bytes); break;
      default: jacobi_sq_launch<448, 7>(c, in, U, s, Vt, tol, bytes); break;
    }
    return;
  }
  // past one CTA's shared memory the scalar kernel would run out of global memory: the block
  // Jacobi is 2-4.5x faster there (n = 128..159: 13.8 / 21.7 / 44.0 -> 7.2 / 8.3 / 9.7 ms,
  // tools/svd_mid.py); below, the single CTA wins (n = 116: 3.9 vs 7.1 ms)
  if ((long long)m * n + (long long)n * n + n > kSmemDoubles) {
    svd_block_jacobi(c, in, U, s, Vt);
    return;
  }
  const int len = std::max(m, n);  // rows of W (m) and of V (n) per lane slice
  if (len <= 4 * 32)
    jacobi_launch<4, 32>(c, in, U, s, Vt, tol);
  else if (len <= 8 * 32)
    jacobi_launch<8, 32>(c, in, U, s, Vt, tol);
  else if (len <= 16 * 32)
    jacobi_launch<16, 32>(c, in, U, s, Vt, tol);
  else if (len <= 32 * 32)
    jacobi_launch<32, 32>(c, in, U, s, Vt, tol);
  else
    svd_block_jacobi(c, in, U, s, Vt);
}

namespace {

// perm = columns of A (m x n) by decreasing 2-norm (stable), one CTA
__global__ void __launch_bounds__(256) sort_cols_kernel(CMatView A, int* perm) {
  extern __shared__ double nrm[];
  const int m = A.rows, n = A.cols;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < n; j += 8) {
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) {
      const double v = A.p[(long long)i * A.rs + (long long)j * A.cs];
      s2 += v * v;
    }
    s2 = warp_sum(s2);
    if (lane == 0) nrm[j] = s2;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += 256) {
    const double v = nrm[j];
    int r = 0;
    for (int d = 0; d < n; ++d) r += (nrm[d] > v) || (nrm[d] == v && d < j);
    perm[r] = j;
  }
}

__global__ void gather_cols_kernel(CMatView A, const int* perm, double* out) {  // out row-major m x n
  const long long total = (long long)A.rows * A.cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / A.cols), j = (int)(e % A.cols);
    out[e] = A.p[(long long)i * A.rs + (long long)perm[j] * A.cs];
  }
}

// Vt[k][perm[j]] = UX[j][k]   (UX n x n row-major)
__global__ void scatter_vt_kernel(const double* UX, const int* perm, int n, MatView Vt) {
  const long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / n), k = (int)(e % n);
    Vt.p[(long long)k * Vt.rs + (long long)perm[j] * Vt.cs] = UX[e];
  }
}

}  // namespace

// SVD of a tall matrix (m >= n) by preconditioned one-sided Jacobi: columns sorted by
// decreasing norm, A P = Q R, then Jacobi on X = R^T (rows graded by the sort), so
// R = V_X S U_X^T and A = (Q V_X) S (P U_X)^T.  On graded truncation matrices this
// takes ~10 sweeps where Jacobi on R took 15-30 (tools/svd_bench.py).
static void svd_tall(Ctx& c, CMatView in, MatView U, double* s, MatView Vt) {
  const int m = in.rows, n = in.cols;
  DBuf permb(cdiv(n, 2) + 1, c.stream), Ap((long long)m * n, c.stream);
  int* perm = reinterpret_cast<int*>(permb.p);
  sort_cols_kernel<<<1, 256, n * sizeof(double), c.stream>>>(in, perm);
  QTT_CHECK_LAUNCH();
  gather_cols_kernel<<<grid_for((long long)m * n), 256, 0, c.stream>>>(in, perm, Ap.p);
  QTT_CHECK_LAUNCH();
  DBuf Q((long long)m * n, c.stream), R((long long)n * n, c.stream), UX((long long)n * n, c.stream),
      VX((long long)n * n, c.stream);
  qr(c, crowmajor(Ap.p, m, n), rowmajor(Q.p, m, n), rowmajor(R.p, n, n));
  // Jacobi on R^T (block one-sided Jacobi over all CTAs past one CTA's reach): UX (n x n) and V_X written untransposed into VX (row-major [i][rank])
  jacobi(c, ctrans(crowmajor(R.p, n, n)), rowmajor(UX.p, n, n), s, trans(rowmajor(VX.p, n, n)));
  if (U.p) {  // U = Q V_X
    GemmArgs g;
    g.M = m; g.N = n; g.K = n;
    gemm_set_A(g, Q.p, n, false);
    gemm_set_B(g, VX.p, n, false);
    g.C = U.p; g.c_rs = U.rs; g.c_cs = U.cs;
    gemm(g, c.stream);
  }
  if (Vt.p) {
    scatter_vt_kernel<<<grid_for((long long)n * n), 256, 0, c.stream>>>(UX.p, perm, n, Vt);
    QTT_CHECK_LAUNCH();
  }
}

void svd(Ctx& c, CMatView in, MatView U, double* s, MatView Vt) {
  const int m = in.rows, n = in.cols;
  if (m <= 0 || n <= 0) return;
  c.stats.svd_calls++;
  if (m >= n)
    svd_tall(c, in, U, s, Vt);
  else  // in^T = U' S V'^T  =>  in = V' S U'^T
    svd_tall(c, ctrans(in), trans(Vt), s, trans(U));
}

void potrf_lower(Ctx& c, double* A, int dim, long long ld, int* info) {
  QTT_CUDA(cudaMemsetAsync(info, 0, sizeof(int), c.stream));
  for (int j0 = 0; j0 < dim; j0 += CB) {
    const int nb = std::min(CB, dim - j0);
    potrf_diag_kernel<<<1, 256, 0, c.stream>>>(A, dim, ld, j0, info);
    QTT_CHECK_LAUNCH();
    const int rest = dim - j0 - nb;
    if (rest <= 0) break;
    potrf_trsm_kernel<<<cdiv(rest, 128), 128, 0, c.stream>>>(A, dim, ld, j0, info);
    QTT_CHECK_LAUNCH();
    GemmArgs g;  // A22 -= L21 L21^T  (lower tiles only)
    g.M = rest; g.N = rest; g.K = nb;
    double* L21 = A + (long long)(j0 + nb) * ld + j0;
    gemm_set_A(g, L21, ld, false);
    gemm_set_B(g, L21, ld, true);
    gemm_set_C(g, A + (long long)(j0 + nb) * ld + j0 + nb, ld);
    g.alpha = -1.0; g.beta = 1.0;
    g.lower_only = true;
    g.skip = info;
    gemm(g, c.stream);
  }
  c.stats.chol_solves++;
}

namespace {
__global__ void add_diag_kernel(double* A, int n, long long ld, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) A[(long long)i * ld + i] += v;
}
}  // namespace

void add_diag(Ctx& c, double* A, int n, long long ld, double v) {
  add_diag_kernel<<<cdiv(n, 256), 256, 0, c.stream>>>(A, n, ld, v);
  QTT_CHECK_LAUNCH();
}

void potrs_lower(Ctx& c, const double* L, int dim, long long ld, double* b) {
  potrs_kernel<<<1, 1024, 0, c.stream>>>(L, dim, ld, b);
  QTT_CHECK_LAUNCH();
}

void max_abs_row_sum(Ctx& c, const double* A, int dim, long long ld, double* out) {
  QTT_CUDA(cudaMemsetAsync(out, 0, sizeof(double), c.stream));
  row_abs_sum_kernel<<<cdiv((long long)dim * 32, 256), 256, 0, c.stream>>>(A, dim, ld, out);
  QTT_CHECK_LAUNCH();
}

void dot(Ctx& c, const double* a, const double* b, long long n, double* out) { reduce<0>(c, a, b, n, out); }
void sum(Ctx& c, const double* a, long long n, double* out) { reduce<1>(c, a, nullptr, n, out); }
void nrm2(Ctx& c, const double* a, long long n, double* out) { reduce<2>(c, a, nullptr, n, out); }

void read_scalars(Ctx& c, const double* dev, int n, double* host) {
  double* pin = c.host_scalars(n);
  QTT_CUDA(cudaMemcpyAsync(pin, dev, n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  for (int i = 0; i < n; ++i) host[i] = pin[i];
}

void kron_core(Ctx& c, const double* A, int Ra0, int m, int n, int Ra1, const double* x, int rx0,
               int rx1, double* y) {
  const long long total = (long long)Ra0 * rx0 * m * Ra1 * rx1;
  const long long rows = (long long)Ra0 * rx0 * m;
  const size_t sh = (size_t)n * (Ra1 + rx1) * sizeof(double);
  const int staged = sh <= 48 * 1024 ? 1 : 0;
  (void)total;
  kron_core_kernel<<<(int)std::min<long long>(rows, 148LL * 16), 256, staged ? sh : 0, c.stream>>>(
      A, Ra0, m, n, Ra1, x, rx0, rx1, y, staged);
  QTT_CHECK_LAUNCH();
}

namespace {
// All Kronecker cores of a TT-matvec in one launch (tt.py:443-447): global output row g of the
// concatenated cores -> (core k: desc row0 <= g, row (a, xx, mm) of that core).  One WARP per
// row (no block barriers: 8 independent write streams per CTA), the A and x slices read through
// L1, the row (Ra1 * rx1 contiguous doubles) written with 16-byte streaming stores -- a pure HBM
// write stream across all cores, no per-core launch gaps or tails.
__global__ void __launch_bounds__(256) kron_all_kernel(const KronDesc* __restrict__ desc, int K,
                                                       long long rows_total) {
  __shared__ KronDesc sd[kKronMaxCores];
  for (int i = threadIdx.x; i < K; i += blockDim.x) sd[i] = desc[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows_total;
       row += nw) {
    int lo = 0, hi = K - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sd[mid].row0 <= row) lo = mid; else hi = mid - 1;
    }
    const KronDesc& d = sd[lo];
    const long long r = row - d.row0;
    const int m = d.m, n = d.n, Ra1 = d.Ra1, rx1 = d.rx1;
    const int mm = (int)(r % m);
    const long long t = r / m;
    const int xx = (int)(t % d.rx0), a = (int)(t / d.rx0);
    const double* sa = d.A + ((long long)a * m + mm) * n * Ra1;
    const double* sx = d.x + (long long)xx * n * rx1;
    const int cols = Ra1 * rx1;
    double* yr = d.y + r * cols;
    if ((rx1 & 1) == 0) {
      const int h = rx1 >> 1;
      double2* dst = reinterpret_cast<double2*>(yr);
      for (int e = lane; e < Ra1 * h; e += 32) {
        const int b = e / h, j = e - b * h;
        double s0 = 0.0, s1 = 0.0;
        for (int nn = 0; nn < n; ++nn) {
          const double av = __ldg(sa + nn * Ra1 + b);
          const double2 xv = __ldg(reinterpret_cast<const double2*>(sx + nn * rx1) + j);
          s0 = fma(av, xv.x, s0);
          s1 = fma(av, xv.y, s1);
        }
        __stcs(dst + e, make_double2(s0, s1));
      }
    } else {
      for (int e = lane; e < cols; e += 32) {
        const int b = e / rx1, yy = e - b * rx1;
        double sum = 0.0;
        for (int nn = 0; nn < n; ++nn) sum += __ldg(sa + nn * Ra1 + b) * __ldg(sx + nn * rx1 + yy);
        __stcs(yr + e, sum);
      }
    }
  }
}
}  // namespace

void kron_all(Ctx& c, const std::vector<KronDesc>& cores) {
  const int K = (int)cores.size();
  if (K == 0) return;
  if (K > kKronMaxCores) throw Error(QTT_ERR_ARG, "kron_all: too many cores");
  std::vector<KronDesc> d(cores);
  long long rows = 0;
  bool aligned = true;
  for (auto& e : d) {
    e.row0 = rows;
    rows += (long long)e.Ra0 * e.rx0 * e.m;
    if ((e.rx1 & 1) == 0 && ((reinterpret_cast<uintptr_t>(e.x) | reinterpret_cast<uintptr_t>(e.y)) & 15) != 0)
      aligned = false;
  }
  if (!aligned) throw Error(QTT_ERR_ARG, "kron_all: cores must be 16-byte aligned");
  // (a pageable source: the copy is staged before cudaMemcpyAsync returns, d may go out of scope)
  DBuf dd((long long)((K * sizeof(KronDesc) + 7) / 8), c.stream);
  QTT_CUDA(cudaMemcpyAsync(dd.p, d.data(), K * sizeof(KronDesc), cudaMemcpyHostToDevice, c.stream));
  kron_all_kernel<<<(int)std::min<long long>(cdiv(rows, 8), 148LL * 8), 256, 0, c.stream>>>(
      reinterpret_cast<const KronDesc*>(dd.p), K, rows);
  QTT_CHECK_LAUNCH();
}

void scale_rows(Ctx& c, const double* in, long long ld_in, const double* scale, int rows, int cols,
                double* out, long long ld_out) {
  scale_rows_kernel<<<grid_for((long long)rows * cols), 256, 0, c.stream>>>(in, ld_in, scale, rows,
                                                                            cols, out, ld_out);
  QTT_CHECK_LAUNCH();
}

void copy_view(Ctx& c, CMatView in, MatView out) {
  copy_view_kernel<<<grid_for((long long)in.rows * in.cols), 256, 0, c.stream>>>(in, out);
  QTT_CHECK_LAUNCH();
}

void fill(Ctx& c, double* p, long long n, double v) {
  if (n <= 0) return;
  fill_kernel<<<grid_for(n), 256, 0, c.stream>>>(p, n, v);
  QTT_CHECK_LAUNCH();
}

void axpby(Ctx& c, long long n, double a, const double* x, double b, double* y) {
  axpby_kernel<<<grid_for(n), 256, 0, c.stream>>>(n, a, x, b, y);
  QTT_CHECK_LAUNCH();
}

void op_core_diag(Ctx& c, const double* A, int R0, int m, int R1, double* d) {
  op_core_diag_kernel<<<grid_for((long long)R0 * m * R1), 256, 0, c.stream>>>(A, R0, m, R1, d);
  QTT_CHECK_LAUNCH();
}

}  // namespace qtt
