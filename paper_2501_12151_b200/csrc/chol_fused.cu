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
// CTA; the trailing updates use a 16x16 thread map (no per-element div/mod).
// Returns 0 or the 1-based failing column (global index).
__device__ int factor_diag(double* A, long long ld, int j0, int nb, double* s) {
  for (int e = threadIdx.x; e < nb * nb; e += NT) {
    const int i = e / nb, j = e % nb;
    s[i * LD + j] = (j <= i) ? __ldcg(A + (long long)(j0 + i) * ld + j0 + j) : 0.0;
  }
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  for (int j = 0; j < nb; ++j) {
    const double d = s[j * LD + j];
    if (!(d > 0.0)) {  // dpotrf: non-positive or NaN pivot
      if (threadIdx.x == 0) bad = j0 + j + 1;
      __syncthreads();
      break;
    }
    const double ljj = sqrt(d), inv = 1.0 / ljj;
    // scale column j below the diagonal (rows j+1..nb-1); diagonal written after
    for (int i = j + 1 + threadIdx.x; i < nb; i += NT) s[i * LD + j] *= inv;
    __syncthreads();
    if (threadIdx.x == 0) s[j * LD + j] = ljj;
    for (int i = j + 1 + ty; i < nb; i += 16) {
      const double lij = s[i * LD + j];
      for (int c = j + 1 + tx; c <= i; c += 16) s[i * LD + c] -= lij * s[c * LD + j];
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
// nb x nb block in shared memory s: one thread per column, forward substitution.
__device__ void invert_lower(const double* s, int nb, double* Linv) {
  const int c = threadIdx.x;
  if (c < NB) {
    double x[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      if (i < nb && i >= c) {
#pragma unroll
        for (int p = 0; p < i; ++p)
          if (p >= c) v -= s[i * LD + p] * x[p];
        x[i] = v / s[i * LD + i];
      } else {
        x[i] = 0.0;
      }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) Linv[i * NB + c] = x[i];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NT) chol_fused_kernel(CholArgs a) {
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

  // ---- blocked right-looking Cholesky
  for (int j0 = 0; j0 < dim; j0 += NB) {
    const int nb = min(NB, dim - j0);
    const int rest = dim - j0 - nb;
    if (blockIdx.x == 0) {
      const int b = factor_diag(A, ld, j0, nb, smem);
      if (threadIdx.x == 0 && b != 0) *a.info = b;
    }
    grid.sync();
    mark(1);
    if (__ldcg(a.info) != 0) return;  // uniform: every CTA reads the same flag
    if (rest <= 0) break;
    // panel solve: L21 = A21 L11^-T, one thread per row, L11 staged in shared memory
    {
      double* L = smem;
      for (int e = threadIdx.x; e < nb * nb; e += NT) {
        const int i = e / nb, j = e % nb;
        L[i * LD + j] = (j <= i) ? __ldcg(A + (long long)(j0 + i) * ld + j0 + j) : 0.0;
      }
      __syncthreads();
      for (int row = j0 + nb + blockIdx.x * NT + threadIdx.x; row < dim; row += gridDim.x * NT) {
        double x[NB];
        double* ar = A + (long long)row * ld + j0;
#pragma unroll
        for (int j = 0; j < NB; ++j) x[j] = j < nb ? ar[j] : 0.0;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          if (j < nb) {
            double v = x[j];
#pragma unroll
            for (int p = 0; p < j; ++p) v -= x[p] * L[j * LD + p];
            x[j] = v / L[j * LD + j];
          }
        }
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (j < nb) ar[j] = x[j];
      }
      __syncthreads();
    }
    grid.sync();
    mark(2);
    // trailing update  A22 -= L21 L21^T  on lower tiles (DMMA)
    {
      const double* L21 = A + (long long)(j0 + nb) * ld + j0;
      double* A22 = A + (long long)(j0 + nb) * ld + j0 + nb;
      const int tiles = (rest + NB - 1) / NB;
      const int items = tiles * (tiles + 1) / 2;
      tile::Operands o{L21, ld, 1, L21, 1, ld, rest, rest, nb};
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
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
      }
    }
    grid.sync();
    mark(3);
  }

  // ---- invert every diagonal block (in parallel over CTAs)
  for (int bk = blockIdx.x; bk < nblk; bk += gridDim.x) {
    const int j0 = bk * NB, nb = min(NB, dim - j0);
    for (int e = threadIdx.x; e < NB * NB; e += NT) {
      const int i = e / NB, j = e % NB;
      smem[i * LD + j] = (i < nb && j <= i) ? __ldcg(A + (long long)(j0 + i) * ld + j0 + j) : (i == j ? 1.0 : 0.0);
    }
    __syncthreads();
    invert_lower(smem, NB, a.Linv + (long long)bk * NB * NB);
  }
  grid.sync();
  mark(4);

  // ---- forward: L y = b.  Every CTA forms y_j = Linv_j x_j itself (x_j is final
  // once the previous blocks' updates are in), then updates its rows below; y goes to
  // a separate buffer so no CTA overwrites an x_j another CTA is still reading.
  double* x = a.x;
  double* y = a.y;
  for (int bk = 0; bk < nblk; ++bk) {
    const int j0 = bk * NB, nb = min(NB, dim - j0);
    const double* Li = a.Linv + (long long)bk * NB * NB;
    if (warp < 2) {  // 64 rows of the 64x64 product, one row per thread of warps 0-1
      const int i = threadIdx.x;
      double s = 0.0;
      for (int j = 0; j <= i && j < nb; ++j) s += __ldcg(Li + i * NB + j) * __ldcg(x + j0 + j);
      yb[i] = i < nb ? s : 0.0;
    }
    __syncthreads();
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < nb; i += NT) y[j0 + i] = yb[i];
    for (int row = j0 + nb + gwarp; row < dim; row += nwarps) {  // one warp per row
      double s = 0.0;
      for (int j = lane; j < nb; j += 32) s += A[(long long)row * ld + j0 + j] * yb[j];
      s = warp_sum(s);
      if (lane == 0) x[row] -= s;
    }
    grid.sync();
  }
  mark(5);
  // ---- backward: L^T u = y, blocks last to first: u_j = Linv_j^T y_j (y is the
  // working vector, updated above the block; u is written to x)
  for (int bk = nblk - 1; bk >= 0; --bk) {
    const int j0 = bk * NB, nb = min(NB, dim - j0);
    const double* Li = a.Linv + (long long)bk * NB * NB;
    if (warp < 2) {
      const int i = threadIdx.x;
      double s = 0.0;
      for (int j = i; j < nb; ++j) s += __ldcg(Li + j * NB + i) * __ldcg(y + j0 + j);  // (Linv^T)[i][j]
      yb[i] = i < nb ? s : 0.0;
    }
    __syncthreads();
    if (blockIdx.x == 0)
      for (int i = threadIdx.x; i < nb; i += NT) x[j0 + i] = yb[i];
    // y[i] -= sum_j L[j0+j, i] u[j] for i < j0 (coalesced over i)
    for (int i = blockIdx.x * NT + threadIdx.x; i < j0; i += gridDim.x * NT) {
      double s = 0.0;
      for (int j = 0; j < nb; ++j) s += A[(long long)(j0 + j) * ld + i] * yb[j];
      y[i] -= s;
    }
    grid.sync();
  }
}

}  // namespace

int chol_fused_grid(int device) {
  static int cached = -1;
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
