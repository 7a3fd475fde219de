// Direct local solve (amen.py:181-191) as ONE persistent cooperative kernel:
//   lam = max_i sum_j |M_ij|                      (Gershgorin bound, amen.py:190)
//   M = L L^T  blocked right-looking, NB = 64     (scipy cho_factor(lower=True) / dpotrf)
//   u = L^-T L^-1 b                               (cho_solve / dpotrs)
// Phases are separated by grid-wide barriers: the 64x64 diagonal factor runs in one
// CTA (shared memory, 2D thread map), the panel solve over all CTAs (one row per
// thread), the trailing update as DMMA tiles (dmma_tile.cuh).  The triangular solves
// use inverted 64x64 diagonal blocks (all inverted in parallel after the
// factorization) so every CTA can form each block's solution itself: one barrier
// per block and direction.  A non-positive (or NaN) pivot stops the factorization
// with info = j+1, exactly LAPACK's rule, and the host raises the reference's SolverError.
#include <cooperative_groups.h>

#include <algorithm>

#include "chol_fused.cuh"
#include "dmma_tile.cuh"

namespace cg = cooperative_groups;

namespace qtt {
namespace {

using CF = tile::Cfg<64, 64, 16, 2, 4, 3>;  // 256 threads
constexpr int NT = CF::NT;
constexpr int NB = 64;
constexpr int LD = NB + 1;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Factor the nb x nb diagonal block at (j0, j0) in shared memory s (stride LD), one
// CTA, blocked by PW = 8 columns: warp 0 factors each 8-column panel (rows k0..nb-1, two
// rows per lane, warp-synchronous: pivots and multipliers travel by shuffles, no block
// barrier), then all threads apply the rank-8 update to the trailing lower triangle.
// Returns 0 or the 1-based failing column (global index).
__device__ int factor_diag(double* A, long long ld, int j0, int nb, double* s) {
  constexpr int PW = 8;
  for (int e = threadIdx.x; e < nb * nb; e += NT) {
    const int i = e / nb, j = e % nb;
    s[i * LD + j] = (j <= i) ? __ldcg(A + (long long)(j0 + i) * ld + j0 + j) : 0.0;
  }
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  for (int k0 = 0; k0 < nb; k0 += PW) {
    const int pw = min(PW, nb - k0);
    if (warp == 0) {
      const int ra = k0 + lane, rb = k0 + 32 + lane;  // this lane's panel rows
      double v[2][PW];
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        v[0][c] = (ra < nb && c < pw) ? s[ra * LD + k0 + c] : 0.0;
        v[1][c] = (rb < nb && c < pw) ? s[rb * LD + k0 + c] : 0.0;
      }
      int fail = 0;
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        if (c < pw && fail == 0) {
          const double d = __shfl_sync(0xffffffffu, v[0][c], c);  // row k0 + c lives in lane c
          if (!(d > 0.0)) {
            fail = j0 + k0 + c + 1;  // dpotrf: non-positive or NaN pivot
          } else {
            const double l = sqrt(d), inv = 1.0 / l;
            if (ra > k0 + c) v[0][c] *= inv;
            if (ra == k0 + c) v[0][c] = l;
            if (rb < nb) v[1][c] *= inv;
#pragma unroll
            for (int c2 = c + 1; c2 < PW; ++c2) {
              const double m = __shfl_sync(0xffffffffu, v[0][c], c2);  // L[k0 + c2][c]
              if (c2 < pw) {
                if (ra >= k0 + c2) v[0][c2] = fma(-v[0][c], m, v[0][c2]);
                if (rb < nb) v[1][c2] = fma(-v[1][c], m, v[1][c2]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        if (c < pw) {
          if (ra < nb && ra >= k0 + c) s[ra * LD + k0 + c] = v[0][c];
          if (rb < nb) s[rb * LD + k0 + c] = v[1][c];
        }
      }
      if (lane == 0 && fail != 0) bad = fail;
    }
    __syncthreads();
    if (bad != 0) break;  // uniform
    // rank-pw update of the trailing lower triangle: rows/cols >= k0 + pw
    const int t0 = k0 + pw;
    for (int i = t0 + ty; i < nb; i += 16) {
      double li[PW];
#pragma unroll
      for (int c = 0; c < PW; ++c) li[c] = c < pw ? s[i * LD + k0 + c] : 0.0;
      for (int jc = t0 + tx; jc <= i; jc += 16) {
        double acc = s[i * LD + jc];
#pragma unroll
        for (int c = 0; c < PW; ++c) acc = fma(-li[c], s[jc * LD + k0 + c], acc);
        s[i * LD + jc] = acc;
      }
    }
    __syncthreads();
  }
  const int b = bad;
  if (b == 0)
    for (int e = threadIdx.x; e < nb * nb; e += NT) {
      const int i = e / nb, j = e % nb;
      if (j <= i) A[(long long)(j0 + i) * ld + j0 + j] = s[i * LD + j];
    }
  __syncthreads();
  return b;
}

// Linv (NB x NB row-major, zero above the diagonal) = inverse of the lower-triangular
// nb x nb block in shared memory s: forward substitution, 4 lanes per column (each lane
// owns every 4th row of the column's solution in registers; the partial dot products of
// a row are combined with two shuffles).  Requires NT == 4 * NB.
__device__ void invert_lower(const double* s, int nb, double* Linv) {
  static_assert(NT == 4 * NB, "4 lanes per column");
  __shared__ double rdiag[NB];
  if (threadIdx.x < NB) rdiag[threadIdx.x] = threadIdx.x < nb ? 1.0 / s[threadIdx.x * LD + threadIdx.x] : 0.0;
  __syncthreads();
  const int c = threadIdx.x >> 2, part = threadIdx.x & 3;
  double xs[NB / 4];
#pragma unroll
  for (int k = 0; k < NB / 4; ++k) xs[k] = 0.0;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    double a0 = 0.0, a1 = 0.0;  // two independent FMA chains
#pragma unroll
    for (int k = 0; k < NB / 4; k += 2) {
      const int p0 = part + 4 * k, p1 = p0 + 4;
      if (p0 < i && p0 >= c) a0 = fma(s[i * LD + p0], xs[k], a0);
      if (p1 < i && p1 >= c) a1 = fma(s[i * LD + p1], xs[k + 1], a1);
    }
    double acc = a0 + a1;
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    double xi = 0.0;
    if (i < nb && i >= c) xi = ((i == c ? 1.0 : 0.0) - acc) * rdiag[i];
    if (part == (i & 3)) xs[i >> 2] = xi;
  }
#pragma unroll
  for (int k = 0; k < NB / 4; ++k) Linv[(part + 4 * k) * NB + c] = xs[k];
  __syncthreads();
}

__global__ void __launch_bounds__(NT, 1) chol_fused_kernel(CholArgs a) {
  extern __shared__ double smem[];
  __shared__ double yb[NB];
  cg::grid_group grid = cg::this_grid();
  unsigned long long tp = gtimer();
  auto mark = [&](int ph) {
    if (a.phase_ns != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
      const unsigned long long now = gtimer();
      a.phase_ns[ph] += now - tp;
      tp = now;
    }
  };
  double* A = a.A;
  const int dim = a.dim;
  const long long ld = a.ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * (NT / 32) + warp, nwarps = gridDim.x * (NT / 32);
  const int nblk = (dim + NB - 1) / NB;

  // ---- lam = max abs row sum of the original matrix (one warp per row; L2-only loads)
  for (int row = gwarp; row < dim; row += nwarps) {
    double s = 0.0;
    for (int j = lane; j < dim; j += 32) s += fabs(__ldcg(A + (long long)row * ld + j));
    s = warp_sum(s);
    if (lane == 0) atomicMax((unsigned long long*)a.lam, (unsigned long long)__double_as_longlong(s));
  }
  grid.sync();
  mark(0);

  // ---- blocked right-looking Cholesky with look-ahead.  Step j: (panel) every CTA forms
  // L21 = A21 Linv_j^T for its 64-row blocks as DMMA tiles (Linv_j = L11^-1 from the
  // diagonal factor), barrier, (trailing) A22 -= L21 L21^T on the lower tiles -- and CTA 0
  // first updates the NEXT diagonal tile and factors + inverts it right away, so the next
  // step's diagonal factor overlaps this step's trailing update instead of running alone.
  if (blockIdx.x == 0) {
    const int b = factor_diag(A, ld, 0, min(NB, dim), smem);
    if (threadIdx.x == 0 && b != 0) *a.info = b;
    mark(1);
    if (b == 0) invert_lower(smem, min(NB, dim), a.Linv);
    mark(4);
  }
  grid.sync();
  for (int j0 = 0; j0 < dim; j0 += NB) {
    if (__ldcg(a.info) != 0) return;  // uniform: every CTA reads the same flag
    const int bk = j0 / NB;
    const int nb = min(NB, dim - j0);
    const int rest = dim - j0 - nb;
    if (rest <= 0) break;
    // panel: L21 = A21 Linv^T  (B(k, n) = Linv[n][k])
    {
      const double* Li = a.Linv + (long long)bk * NB * NB;
      double* A21 = A + (long long)(j0 + nb) * ld + j0;
      const int rtiles = (rest + NB - 1) / NB;
      tile::Operands o{A21, ld, 1, Li, 1, NB, rest, nb, nb};
      for (int t = blockIdx.x; t < rtiles; t += gridDim.x) {
        double acc[CF::MI][CF::NI][2];
        tile::zero_acc<CF>(acc);
        tile::mma_tile<CF>(o, t * NB, 0, 0, (nb + CF::BK - 1) / CF::BK, smem, acc);
        tile::for_each_acc<CF>(t * NB, 0, rest, nb, acc,
                               [&](int r, int c, double v) { A21[(long long)r * ld + c] = v; });
      }
    }
    grid.sync();
    mark(2);
    // trailing update  A22 -= L21 L21^T  on lower tiles (DMMA); item 0 = next diagonal tile
    {
      const double* L21 = A + (long long)(j0 + nb) * ld + j0;
      double* A22 = A + (long long)(j0 + nb) * ld + j0 + nb;
      const int tiles = (rest + NB - 1) / NB;
      const int items = tiles * (tiles + 1) / 2;
      tile::Operands o{L21, ld, 1, L21, 1, ld, rest, rest, nb};
      auto do_item = [&](int it) {
        // it -> (ti, tj) with tj <= ti (row-major over the lower triangle of tiles)
        int ti = (int)((sqrt(8.0 * it + 1.0) - 1.0) / 2.0);
        while ((ti + 1) * (ti + 2) / 2 <= it) ++ti;
        while (ti * (ti + 1) / 2 > it) --ti;
        const int tj = it - ti * (ti + 1) / 2;
        double acc[CF::MI][CF::NI][2];
        tile::zero_acc<CF>(acc);
        tile::mma_tile<CF>(o, ti * NB, tj * NB, 0, (nb + CF::BK - 1) / CF::BK, smem, acc);
        tile::for_each_acc<CF>(ti * NB, tj * NB, rest, rest, acc, [&](int r, int c, double v) {
          if (c <= r) A22[(long long)r * ld + c] -= v;
        });
      };
      if (blockIdx.x == 0) {
        do_item(0);
        __threadfence_block();
        __syncthreads();
        const int nb2 = min(NB, rest);
        const int b = factor_diag(A, ld, j0 + nb, nb2, smem);
        if (threadIdx.x == 0 && b != 0) *a.info = b;
        if (b == 0) invert_lower(smem, nb2, a.Linv + (long long)(bk + 1) * NB * NB);
      }
      const int G1 = gridDim.x > 1 ? gridDim.x - 1 : 1;
      const int me = gridDim.x > 1 ? (int)blockIdx.x - 1 : 0;
      if (gridDim.x == 1 || blockIdx.x > 0)
        for (int it = 1 + me; it < items; it += G1) do_item(it);
    }
    grid.sync();
    mark(3);
  }

  // ---- triangular solves in groups of GS = 4 diagonal blocks per grid barrier: every CTA
  // solves the group's 256 x 256 diagonal part itself (block by block with the inverted
  // 64 x 64 blocks and the in-group off-diagonal blocks; redundant but tiny), then updates
  // its share of the rows outside the group -- 16 barriers per direction at dim 4096
  // instead of 64.  y goes to a separate buffer so no CTA overwrites an x another still reads.
  constexpr int GS = 4;
  __shared__ double xg[GS * NB];
  double* x = a.x;
  double* y = a.y;
  // forward: L y = b
  for (int bk0 = 0; bk0 < nblk; bk0 += GS) {
    const int g0 = bk0 * NB;
    const int grows = min(GS * NB, dim - g0);
    for (int i = threadIdx.x; i < grows; i += NT) xg[i] = __ldcg(x + g0 + i);
    __syncthreads();
    for (int g = 0; g < GS && bk0 + g < nblk; ++g) {
      const int bk = bk0 + g, j0 = bk * NB, nb = min(NB, dim - j0);
      const double* Li = a.Linv + (long long)bk * NB * NB;
      {  // y_g = Linv_g x_g: 4 lanes per row, 16 independent loads in flight per lane
        const int i = threadIdx.x >> 2, part = threadIdx.x & 3;
        double lv[NB / 4];
#pragma unroll
        for (int k = 0; k < NB / 4; ++k) {
          const int jj = part + 4 * k;
          lv[k] = (jj <= i && jj < nb) ? __ldcg(Li + i * NB + jj) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < NB / 4; ++k) s = fma(lv[k], xg[g * NB + part + 4 * k], s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (part == 0) yb[i] = i < nb ? s : 0.0;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < nb; i += NT) xg[g * NB + i] = yb[i];  // xg now holds y_g
      // in-group rows below: x[r] -= L[r, block g] y_g   (one warp per row)
      for (int r = j0 + nb + warp; r < g0 + grows; r += NT / 32) {
        double t = 0.0;
        for (int jj = lane; jj < nb; jj += 32) t = fma(A[(long long)r * ld + j0 + jj], yb[jj], t);
        t = warp_sum(t);
        if (lane == 0) xg[r - g0] -= t;
      }
      __syncthreads();
    }
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < grows; i += NT) y[g0 + i] = xg[i];
    // rows below the group: x[row] -= L[row, group] y_group   (one warp per row)
    for (int row = g0 + grows + gwarp; row < dim; row += nwarps) {
      double av[GS * NB / 32];
#pragma unroll
      for (int k = 0; k < GS * NB / 32; ++k) {
        const int jj = lane + 32 * k;
        av[k] = jj < grows ? A[(long long)row * ld + g0 + jj] : 0.0;
      }
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < GS * NB / 32; ++k) t = fma(av[k], lane + 32 * k < grows ? xg[lane + 32 * k] : 0.0, t);
      t = warp_sum(t);
      if (lane == 0) x[row] -= t;
    }
    grid.sync();
  }
  mark(5);
  // backward: L^T u = y, groups last to first (y is the working vector; u is written to x)
  const int ngrp = (nblk + GS - 1) / GS;
  for (int gi = ngrp - 1; gi >= 0; --gi) {
    const int bk0 = gi * GS, g0 = bk0 * NB;
    const int grows = min(GS * NB, dim - g0);
    const int nbg = min(GS, nblk - bk0);
    for (int i = threadIdx.x; i < grows; i += NT) xg[i] = __ldcg(y + g0 + i);
    __syncthreads();
    for (int g = nbg - 1; g >= 0; --g) {
      const int bk = bk0 + g, j0 = bk * NB, nb = min(NB, dim - j0);
      const double* Li = a.Linv + (long long)bk * NB * NB;
      {  // u_g = Linv_g^T y_g: 4 lanes per row, 16 independent loads in flight per lane
        const int i = threadIdx.x >> 2, part = threadIdx.x & 3;
        double lv[NB / 4];
#pragma unroll
        for (int k = 0; k < NB / 4; ++k) {
          const int jj = part + 4 * k;
          lv[k] = (jj >= i && jj < nb) ? __ldcg(Li + jj * NB + i) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < NB / 4; ++k) s = fma(lv[k], xg[g * NB + part + 4 * k], s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (part == 0) yb[i] = i < nb ? s : 0.0;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < nb; i += NT) xg[g * NB + i] = yb[i];  // xg now holds u_g
      // in-group columns above: y[c] -= sum_j L[j0 + j, c] u_g[j]   for g0 <= c < j0
      for (int cidx = g0 + threadIdx.x; cidx < j0; cidx += NT) {
        double t = 0.0;
        for (int j16 = 0; j16 < nb; j16 += 16) {
          double av[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) av[k] = j16 + k < nb ? A[(long long)(j0 + j16 + k) * ld + cidx] : 0.0;
#pragma unroll
          for (int k = 0; k < 16; ++k) t = fma(av[k], j16 + k < nb ? yb[j16 + k] : 0.0, t);
        }
        xg[cidx - g0] -= t;
      }
      __syncthreads();
    }
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < grows; i += NT) x[g0 + i] = xg[i];
    // rows above the group: y[i] -= sum_{j in group} L[j, i] u[j]  (coalesced over i)
    for (int i = blockIdx.x * NT + threadIdx.x; i < g0; i += gridDim.x * NT) {
      double t = 0.0;
      for (int j16 = 0; j16 < grows; j16 += 16) {
        double av[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) av[k] = j16 + k < grows ? A[(long long)(g0 + j16 + k) * ld + i] : 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) t = fma(av[k], j16 + k < grows ? xg[j16 + k] : 0.0, t);
      }
      y[i] -= t;
    }
    grid.sync();
  }
}

}  // namespace

int chol_fused_grid(int device) {
  static PerDevice<int> cache(-1);
  int& cached = cache.at(device);
  if (cached > 0) return cached;
  QTT_CUDA(cudaFuncSetAttribute(chol_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM));
  int per_sm = 0, sms = 0;
  QTT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chol_fused_kernel, NT, CF::SMEM));
  QTT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  cached = std::max(1, std::min(per_sm, 1)) * sms;
  return cached;
}

long long chol_fused_linv_doubles(int dim) { return (long long)((dim + NB - 1) / NB) * NB * NB; }

void chol_fused_launch(const CholArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  QTT_CUDA(cudaLaunchCooperativeKernel((void*)chol_fused_kernel, dim3(grid), dim3(NT), args, CF::SMEM, s));
  QTT_CHECK_LAUNCH();
}

}  // namespace qtt
