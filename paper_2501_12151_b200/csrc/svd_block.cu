// Large dense factorizations for rounding-size unfoldings (tt.py:376-406 at bond ranks of
// R*r, e.g. 4096 at config 4): a multi-CTA QR with LAPACK's Q (geqrf_blocked + orgqr_blocked)
// and a block one-sided Jacobi SVD.
//
// Block Jacobi: the columns of B (rows x cols, column-major) are split into blocks of BS;
// a sweep is a round-robin tournament over block pairs (nblk - 1 rounds, all pairs of a
// round in parallel, one CTA each).  For a pair S = I u J the CTA forms G = B_S^T B_S
// (2BS x 2BS), diagonalises it with cyclic two-sided Jacobi in shared memory (G = Z L Z^T),
// and applies Z to the pair's columns of B and of the accumulated V.  A pair counts as
// converged when every |G_pq| <= tol sqrt(G_pp G_qq) or sits at the rounding floor
// eps * max(G_pp, G_qq); the sweep loop ends when a whole sweep rotated nothing.  Column
// norms of the final B are the singular values (absolute accuracy eps * sigma_max, the
// same class as LAPACK gesdd which the reference calls, tt.py:376-383).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "gemm.cuh"
#include "linalg.cuh"
#include "qr_blocked.cuh"
#include "svd_block.cuh"

namespace cg = cooperative_groups;

namespace qtt {
namespace {

constexpr int BJ_NT = 256;
constexpr int BJ_CHUNK = 256;  // rows per staged tile (double-buffered: ~64 KB in flight per SM)

struct BJArgs {
  double* B;        // rows x ncols (column-major, ld = rows), ncols = nblk * BS (zero padded)
  int rows;
  double* V;        // ncols x ncols (column-major), accumulated rotations
  int nblk;
  double tol;       // relative off-diagonal threshold
  int max_sweeps;
  double stop;      // a sweep whose largest relative off-diagonal is <= stop ends the loop
  unsigned long long* offmax;  // [max_sweeps] largest relative off-diagonal seen (double bits)
  int* sweeps_out;
};

__device__ __forceinline__ void pair_of(int round, int i, int nblk, int& I, int& J) {
  // circle method: player nblk-1 fixed, the others rotate
  const int n1 = nblk - 1;
  if (i == 0) {
    I = round;
    J = n1;
  } else {
    I = (round + i) % n1;
    J = (round - i + n1) % n1;
  }
  if (I > J) {
    const int t = I;
    I = J;
    J = t;
  }
}

// columns of the pair: local c < BS -> block I, else block J
__device__ __forceinline__ double* pair_col(double* M, long long ld, int I, int J, int c, int BS) {
  return M + ((long long)(c < BS ? I * BS + c : J * BS + (c - BS))) * ld;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// One staged chunk: rows [r0, r0 + BJ_CHUNK) of the pair's P columns of matrix M (ld, rows).
struct Chunk {
  double* M;
  long long ld;
  int rows, r0;
};

// chunk c of the stream "B rows, then (optionally) V rows"
__device__ __forceinline__ Chunk chunk_at(int c, double* B, int brows, double* V, int vrows) {
  const int nb = (brows + BJ_CHUNK - 1) / BJ_CHUNK;
  if (c < nb) return Chunk{B, brows, brows, c * BJ_CHUNK};
  return Chunk{V, vrows, vrows, (c - nb) * BJ_CHUNK};
}

template <int BS>
__device__ __forceinline__ void issue_chunk(const Chunk& ch, int I, int J, double (*tile)[2 * BS + 1]) {
  constexpr int P = 2 * BS;
  const int nr = min(BJ_CHUNK, ch.rows - ch.r0);
  for (int e = threadIdx.x; e < P * BJ_CHUNK; e += BJ_NT) {
    const int c = e / BJ_CHUNK, i = e % BJ_CHUNK;
    const double* col = pair_col(ch.M, ch.ld, I, J, c, BS);
    cp_async8(&tile[i][c], col + ch.r0 + (i < nr ? i : 0), i < nr);
  }
  cp_commit();
}

// G = M_S^T M_S over rows [0, rows) on the DMMA pipe (m8n8k4: lane l holds A[l/4][l%4],
// B[l%4][l/4], C[l/4][2(l%4) + {0,1}]).  P = 32: warp w owns G fragments (w/2, 2(w%2)+{0,1});
// P = 16: warp w owns fragment ((w/2)%2, w%2) over the k-steps of parity w/4.  Chunks are
// double-buffered with cp.async so the next chunk's loads overlap this chunk's DMMAs.
template <int BS>
__device__ void pair_gram(double* M, int rows, int I, int J, double (*G)[2 * BS + 1],
                          double (*tiles)[BJ_CHUNK][2 * BS + 1]) {
  constexpr int P = 2 * BS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  double acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
  const int pb = P == 32 ? (w >> 1) : ((w >> 1) & 1);
  const int qb = P == 32 ? (w & 1) * 2 : (w & 1);
  const int kpar = P == 32 ? 0 : (w >> 2);
  const int n = (rows + BJ_CHUNK - 1) / BJ_CHUNK;
  __syncthreads();
  issue_chunk<BS>(chunk_at(0, M, rows, nullptr, 0), I, J, tiles[0]);
  for (int c = 0; c < n; ++c) {
    if (c + 1 < n) {
      issue_chunk<BS>(chunk_at(c + 1, M, rows, nullptr, 0), I, J, tiles[(c + 1) & 1]);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    double (*tile)[P + 1] = tiles[c & 1];
    if (P == 32) {
#pragma unroll 4
      for (int ks = 0; ks < BJ_CHUNK / 4; ++ks) {
        const double* row = tile[ks * 4 + lc];
        const double a = row[pb * 8 + lr];
        dmma(acc0, a, row[qb * 8 + lr]);
        dmma(acc1, a, row[(qb + 1) * 8 + lr]);
      }
    } else {
#pragma unroll 4
      for (int ks = kpar; ks < BJ_CHUNK / 4; ks += 2) {
        const double* row = tile[ks * 4 + lc];
        dmma(acc0, row[pb * 8 + lr], row[qb * 8 + lr]);
      }
    }
    __syncthreads();
  }
  if (P == 32) {
    G[pb * 8 + lr][qb * 8 + 2 * lc] = acc0[0];
    G[pb * 8 + lr][qb * 8 + 2 * lc + 1] = acc0[1];
    G[pb * 8 + lr][(qb + 1) * 8 + 2 * lc] = acc1[0];
    G[pb * 8 + lr][(qb + 1) * 8 + 2 * lc + 1] = acc1[1];
  } else {
    if (kpar == 0) {
      G[pb * 8 + lr][qb * 8 + 2 * lc] = acc0[0];
      G[pb * 8 + lr][qb * 8 + 2 * lc + 1] = acc0[1];
    }
    __syncthreads();
    if (kpar == 1) {
      G[pb * 8 + lr][qb * 8 + 2 * lc] += acc0[0];
      G[pb * 8 + lr][qb * 8 + 2 * lc + 1] += acc0[1];
    }
  }
  __syncthreads();
}

// [B_S; V_S] <- [B_S; V_S] Z in one double-buffered chunk stream: per chunk, warp w computes
// output rows [8w, 8w + 8) x all P columns on the DMMA pipe, writes them into the tile, and
// the tile is stored column-coalesced.
template <int BS>
__device__ void pair_update(double* B, int brows, double* V, int vrows, int I, int J,
                            const double (*Z)[2 * BS + 1], double (*tiles)[BJ_CHUNK][2 * BS + 1]) {
  constexpr int P = 2 * BS;
  constexpr int NC = P / 8;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int n = (brows + BJ_CHUNK - 1) / BJ_CHUNK + (vrows + BJ_CHUNK - 1) / BJ_CHUNK;
  __syncthreads();
  issue_chunk<BS>(chunk_at(0, B, brows, V, vrows), I, J, tiles[0]);
  for (int c = 0; c < n; ++c) {
    if (c + 1 < n) {
      issue_chunk<BS>(chunk_at(c + 1, B, brows, V, vrows), I, J, tiles[(c + 1) & 1]);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    double (*tile)[P + 1] = tiles[c & 1];
    constexpr int RG = BJ_CHUNK / (8 * (BJ_NT / 32));  // 8-row groups per warp
    double acc[RG][NC][2];
#pragma unroll
    for (int g = 0; g < RG; ++g)
#pragma unroll
      for (int cb = 0; cb < NC; ++cb) acc[g][cb][0] = acc[g][cb][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < P / 4; ++ks) {
      double zf[NC];
#pragma unroll
      for (int cb = 0; cb < NC; ++cb) zf[cb] = Z[ks * 4 + lc][cb * 8 + lr];
#pragma unroll
      for (int g = 0; g < RG; ++g) {
        const double a = tile[(g * (BJ_NT / 32) + w) * 8 + lr][ks * 4 + lc];
#pragma unroll
        for (int cb = 0; cb < NC; ++cb) dmma(acc[g][cb], a, zf[cb]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < RG; ++g)
#pragma unroll
      for (int cb = 0; cb < NC; ++cb) {
        const int row = (g * (BJ_NT / 32) + w) * 8 + lr;
        tile[row][cb * 8 + 2 * lc] = acc[g][cb][0];
        tile[row][cb * 8 + 2 * lc + 1] = acc[g][cb][1];
      }
    __syncthreads();
    const Chunk ch = chunk_at(c, B, brows, V, vrows);
    const int nr = min(BJ_CHUNK, ch.rows - ch.r0);
    for (int e = threadIdx.x; e < P * BJ_CHUNK; e += BJ_NT) {
      const int cc = e / BJ_CHUNK, i = e % BJ_CHUNK;
      if (i < nr) pair_col(ch.M, ch.ld, I, J, cc, BS)[ch.r0 + i] = tile[i][cc];
    }
    __syncthreads();
  }
}

__device__ __forceinline__ bool needs_rot(double gpp, double gqq, double gpq, double tol) {
  const double a = fabs(gpq);
  if (a == 0.0) return false;
  if (a <= tol * sqrt(gpp) * sqrt(gqq)) return false;
  if (a <= 4.0 * 2.220446049250313e-16 * fmax(gpp, gqq)) return false;  // rounding floor
  return true;
}

// Two-sided cyclic Jacobi on the symmetric P x P matrix G (shared), Z <- eigenvectors.
// Returns whether any rotation was applied (uniform across the CTA).
template <int BS>
__device__ bool pair_eig(double (*G)[2 * BS + 1], double (*Z)[2 * BS + 1], double tol, double* rc, int* flag) {
  constexpr int P = 2 * BS;
  const int t = threadIdx.x;
  for (int e = t; e < P * P; e += BJ_NT) Z[e / P][e % P] = (e / P == e % P) ? 1.0 : 0.0;
  bool any = false;
  for (int sweep = 0; sweep < 20; ++sweep) {
    if (t == 0) *flag = 0;
    __syncthreads();
    for (int step = 0; step < P - 1; ++step) {
      // rotation parameters for the P/2 disjoint pairs of this step
      if (t < P / 2) {
        int p, q;
        if (t == 0) {
          p = step;
          q = P - 1;
        } else {
          p = (step + t) % (P - 1);
          q = (step - t + P - 1) % (P - 1);
        }
        const double gpp = G[p][p], gqq = G[q][q], gpq = G[p][q];
        double c = 1.0, s = 0.0;
        if (needs_rot(gpp, gqq, gpq, tol)) {
          const double tau = (gqq - gpp) / (2.0 * gpq);
          const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + tt * tt);
          s = tt * c;
          *flag = 1;
        }
        rc[4 * t] = c;
        rc[4 * t + 1] = s;
        reinterpret_cast<int*>(rc)[8 * t + 4] = p;
        reinterpret_cast<int*>(rc)[8 * t + 5] = q;
      }
      __syncthreads();
      // rows: G <- J^T G
      for (int e = t; e < (P / 2) * P; e += BJ_NT) {
        const int k = e / P, j = e % P;
        const double c = rc[4 * k], s = rc[4 * k + 1];
        if (s != 0.0) {
          const int p = reinterpret_cast<int*>(rc)[8 * k + 4], q = reinterpret_cast<int*>(rc)[8 * k + 5];
          const double a = G[p][j], b = G[q][j];
          G[p][j] = c * a - s * b;
          G[q][j] = s * a + c * b;
        }
      }
      __syncthreads();
      // columns: G <- G J, Z <- Z J
      for (int e = t; e < (P / 2) * P; e += BJ_NT) {
        const int k = e / P, i = e % P;
        const double c = rc[4 * k], s = rc[4 * k + 1];
        if (s != 0.0) {
          const int p = reinterpret_cast<int*>(rc)[8 * k + 4], q = reinterpret_cast<int*>(rc)[8 * k + 5];
          double a = G[i][p], b = G[i][q];
          G[i][p] = c * a - s * b;
          G[i][q] = s * a + c * b;
          a = Z[i][p];
          b = Z[i][q];
          Z[i][p] = c * a - s * b;
          Z[i][q] = s * a + c * b;
        }
      }
      __syncthreads();
    }
    const int f = *flag;
    __syncthreads();
    if (!f) break;
    any = true;
  }
  if (any) {  // renormalise Z's columns: hundreds of accumulated rotations would otherwise
              // drift the column norms (and with them every singular value) by ~1e-13 per visit
    if (t < P) {
      double s2 = 0.0;
      for (int i = 0; i < P; ++i) s2 = fma(Z[i][t], Z[i][t], s2);
      const double inv = 1.0 / sqrt(s2);
      for (int i = 0; i < P; ++i) Z[i][t] *= inv;
    }
    __syncthreads();
  }
  return any;
}

template <int BS>
__global__ void __launch_bounds__(BJ_NT) bjacobi_kernel(BJArgs a) {
  constexpr int P = 2 * BS;
  __shared__ double G[P][P + 1];
  __shared__ double Z[P][P + 1];
  extern __shared__ double bj_dyn[];
  double (*tiles)[BJ_CHUNK][P + 1] = reinterpret_cast<double (*)[BJ_CHUNK][P + 1]>(bj_dyn);
  __shared__ double rc[4 * 16];
  __shared__ int flag;
  cg::grid_group grid = cg::this_grid();
  const int npairs = a.nblk / 2;
  const int ncols = a.nblk * BS;
  int sw = 0;
  for (; sw < a.max_sweeps; ++sw) {
    for (int round = 0; round < a.nblk - 1; ++round) {
      for (int pi = blockIdx.x; pi < npairs; pi += gridDim.x) {
        int I, J;
        pair_of(round, pi, a.nblk, I, J);
        pair_gram<BS>(a.B, a.rows, I, J, G, tiles);
        // largest relative off-diagonal of the pair (above the rounding floor)
        double off = 0.0;
        for (int e = threadIdx.x; e < P * P; e += BJ_NT) {
          const int p = e / P, q = e % P;
          if (p < q) {
            const double gpp = G[p][p], gqq = G[q][q], g = fabs(G[p][q]);
            if (g > 4.0 * 2.220446049250313e-16 * fmax(gpp, gqq) && gpp > 0.0 && gqq > 0.0)
              off = fmax(off, g / (sqrt(gpp) * sqrt(gqq)));
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) off = fmax(off, __shfl_xor_sync(0xffffffffu, off, o));
        if ((threadIdx.x & 31) == 0) rc[threadIdx.x >> 5] = off;
        __syncthreads();
        off = 0.0;
        for (int i = 0; i < BJ_NT / 32; ++i) off = fmax(off, rc[i]);
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(a.offmax + sw, __double_as_longlong(off));
        if (off > a.tol && pair_eig<BS>(G, Z, a.tol, rc, &flag)) {
          pair_update<BS>(a.B, a.rows, a.V, ncols, I, J, Z, tiles);
        }
      }
      grid.sync();
    }
    if (__longlong_as_double(*(volatile long long*)(a.offmax + sw)) <= a.stop) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.sweeps_out = sw + 1;
}

// sigma_j = ||B[:, j]||, perm = columns by decreasing sigma (stable); one CTA
__global__ void __launch_bounds__(256) colnorm_sort_kernel(const double* B, int rows, int ncols, double* sig,
                                                           int* perm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < ncols; j += 8) {
    double s2 = 0.0;
    for (int i = lane; i < rows; i += 32) {
      const double v = B[(long long)j * rows + i];
      s2 = fma(v, v, s2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) sig[j] = sqrt(s2);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < ncols; j += 256) {
    const double v = sig[j];
    int r = 0;
    for (int d = 0; d < ncols; ++d) r += (sig[d] > v) || (sig[d] == v && d < j);
    perm[r] = j;
  }
}

// outputs for the first k (sorted) columns: s[kk], U[:, kk] = B[:, perm]/sigma, Vt[kk, :] = V[:, perm]^T
__global__ void bj_outputs_kernel(const double* B, int rows, const double* V, int ncols, int cols, const double* sig,
                                  const int* perm, int k, double* s, MatView U, MatView Vt) {
  const long long tu = (long long)rows * k, tv = (long long)k * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tu + tv + k;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < tu) {
      const int kk = (int)(e / rows), i = (int)(e % rows);
      const int j = perm[kk];
      const double sg = sig[j];
      if (U.p) U.p[(long long)i * U.rs + (long long)kk * U.cs] = sg > 0 ? B[(long long)j * rows + i] / sg : 0.0;
    } else if (e < tu + tv) {
      const long long f = e - tu;
      const int kk = (int)(f / cols), i = (int)(f % cols);
      if (Vt.p) Vt.p[(long long)kk * Vt.rs + (long long)i * Vt.cs] = V[(long long)perm[kk] * ncols + i];
    } else {
      const int kk = (int)(e - tu - tv);
      s[kk] = sig[perm[kk]];
    }
  }
}

__global__ void load_padded_kernel(CMatView in, double* B, int ncols, double* V) {
  // B (rows x ncols col-major) = [in, 0]; V = I (ncols x ncols)
  const long long tb = (long long)in.rows * ncols, tv = (long long)ncols * ncols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tb + tv;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < tb) {
      const int j = (int)(e / in.rows), i = (int)(e % in.rows);
      B[e] = j < in.cols ? in.p[(long long)i * in.rs + (long long)j * in.cs] : 0.0;
    } else {
      const long long f = e - tb;
      V[f] = (f % ncols) == (f / ncols) ? 1.0 : 0.0;
    }
  }
}

__global__ void triu_copy_kernel(const double* W, int m, int k, int n, MatView R) {  // R = triu(W)[:k, :n]
  const long long total = (long long)k * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    R.p[(long long)i * R.rs + (long long)j * R.cs] = j >= i ? W[(long long)j * m + i] : 0.0;
  }
}

inline int grid_for(long long n) { return (int)std::max<long long>(1, std::min<long long>(cdiv(n, 256), 1184)); }

template <int BS>
constexpr size_t bj_dyn_bytes() { return 2ull * BJ_CHUNK * (2 * BS + 1) * sizeof(double); }

template <int BS>
int bjacobi_launch(Ctx& c, BJArgs& a) {
  static PerDevice<int> max_dev(-1);
  int& max_blocks = max_dev.at(c.device);
  if (max_blocks < 0) {
    QTT_CUDA(cudaFuncSetAttribute(bjacobi_kernel<BS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)bj_dyn_bytes<BS>()));
    int per_sm = 0, sms = 0;
    QTT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bjacobi_kernel<BS>, BJ_NT, bj_dyn_bytes<BS>()));
    QTT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    max_blocks = std::max(1, per_sm * sms);
  }
  const int grid = std::min(max_blocks, a.nblk / 2);
  void* args[] = {(void*)&a};
  QTT_CUDA(cudaLaunchCooperativeKernel((void*)bjacobi_kernel<BS>, dim3(grid), dim3(BJ_NT), args, bj_dyn_bytes<BS>(),
                                       c.stream));
  QTT_CHECK_LAUNCH();
  return grid;
}

}  // namespace

void svd_block_jacobi(Ctx& c, CMatView in, MatView U, double* s, MatView Vt) {
  const int rows = in.rows, cols = in.cols;
  const int k = std::min(rows, cols);
  // block size: 16 columns (32-column pairs) unless that leaves too few pairs per round
  const int BS = cols >= 16 * 2 * 48 ? 16 : 8;
  int nblk = (int)cdiv(cols, BS);
  nblk += nblk & 1;
  if (nblk < 2) nblk = 2;
  const int ncols = nblk * BS;
  DBuf B((long long)rows * ncols, c.stream), V((long long)ncols * ncols, c.stream);
  load_padded_kernel<<<grid_for((long long)rows * ncols + (long long)ncols * ncols), 256, 0, c.stream>>>(in, B.p, ncols,
                                                                                                       V.p);
  QTT_CHECK_LAUNCH();
  constexpr int MAXSW = 40;
  DBuf flags(MAXSW + 2, c.stream);
  QTT_CUDA(cudaMemsetAsync(flags.p, 0, (MAXSW + 2) * 8, c.stream));
  BJArgs a;
  a.B = B.p;
  a.rows = rows;
  a.V = V.p;
  a.nblk = nblk;
  a.tol = std::sqrt((double)rows) * 2.220446049250313e-16;
  a.max_sweeps = MAXSW;
  a.stop = 8.0 * a.tol;
  a.offmax = reinterpret_cast<unsigned long long*>(flags.p);
  a.sweeps_out = reinterpret_cast<int*>(flags.p + MAXSW);
  if (BS == 16)
    bjacobi_launch<16>(c, a);
  else
    bjacobi_launch<8>(c, a);
  if (std::getenv("QTT_DEBUG_JACOBI")) {
    int sw = 0;
    unsigned long long offs[MAXSW];
    QTT_CUDA(cudaMemcpyAsync(&sw, a.sweeps_out, 4, cudaMemcpyDeviceToHost, c.stream));
    QTT_CUDA(cudaMemcpyAsync(offs, a.offmax, sizeof(offs), cudaMemcpyDeviceToHost, c.stream));
    QTT_CUDA(cudaStreamSynchronize(c.stream));
    std::fprintf(stderr, "[qtt] block jacobi %dx%d BS %d: %d sweeps, max off:", rows, cols, BS, sw);
    for (int i = 0; i < sw && i < MAXSW; ++i) {
      double d;
      std::memcpy(&d, offs + i, 8);
      std::fprintf(stderr, " %.1e", d);
    }
    std::fprintf(stderr, "\n");
  }
  DBuf sig(ncols, c.stream), permb(cdiv(ncols, 2) + 1, c.stream);
  int* perm = reinterpret_cast<int*>(permb.p);
  colnorm_sort_kernel<<<1, 256, 0, c.stream>>>(B.p, rows, ncols, sig.p, perm);
  QTT_CHECK_LAUNCH();
  bj_outputs_kernel<<<grid_for((long long)rows * k + (long long)k * cols + k), 256, 0, c.stream>>>(
      B.p, rows, V.p, ncols, cols, sig.p, perm, k, s, U, Vt);
  QTT_CHECK_LAUNCH();
}

void qr_large(Ctx& c, CMatView in, MatView Q, MatView R) {
  const int m = in.rows, n = in.cols, k = std::min(m, n);
  DBuf W((long long)m * n, c.stream), tau(k, c.stream);
  copy_view(c, in, MatView{W.p, m, n, 1, m});
  geqrf_blocked(c, W.p, m, n, tau.p);
  if (R.p) {
    triu_copy_kernel<<<grid_for((long long)k * n), 256, 0, c.stream>>>(W.p, m, k, n, R);
    QTT_CHECK_LAUNCH();
  }
  if (Q.p) {
    DBuf Qc((long long)m * k, c.stream);
    orgqr_blocked(c, W.p, m, k, tau.p, Qc.p);
    copy_view(c, CMatView{Qc.p, m, k, 1, m}, Q);
  }
}

}  // namespace qtt
