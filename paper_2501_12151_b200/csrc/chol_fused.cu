// Direct local solve (amen.py:181-191) as ONE persistent cooperative kernel:
//   lam = max_i sum_j |M_ij|                      (Gershgorin bound, amen.py:190)
//   M = L L^T  blocked right-looking, NB = 64     (scipy cho_factor(lower=True) / dpotrf)
//   u = L^-T L^-1 b                               (cho_solve / dpotrs)
// Phases are separated by grid-wide barriers: the 64x64 diagonal factor runs in one
// CTA, the panel solve and the DMMA trailing update (dmma_tile.cuh) over all CTAs,
// the triangular solves block by block.  A non-positive (or NaN) pivot stops the
// factorization with info = j+1, exactly LAPACK's rule, and the host raises the
// reference's SolverError.
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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Factor the nb x nb diagonal block at (j0, j0) in shared memory (one CTA).
// Returns 0 or the 1-based failing column (global index).
__device__ int factor_diag(double* A, long long ld, int j0, int nb, double* s /* NB*(NB+1) */) {
  constexpr int LD = NB + 1;
  for (int e = threadIdx.x; e < nb * nb; e += NT) {
    const int i = e / nb, j = e % nb;
    s[i * LD + j] = (j <= i) ? A[(j0 + i) * ld + j0 + j] : 0.0;
  }
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double d = s[j * LD + j];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) bad = j0 + j + 1;
      __syncthreads();
      break;
    }
    const double ljj = sqrt(d);
    __syncthreads();
    if (threadIdx.x == 0) s[j * LD + j] = ljj;
    for (int i = j + 1 + threadIdx.x; i < nb; i += NT) s[i * LD + j] /= ljj;
    __syncthreads();
    const int rem = nb - j - 1;
    for (int e = threadIdx.x; e < rem * rem; e += NT) {
      const int i = j + 1 + e / rem, c = j + 1 + e % rem;
      if (c <= i) s[i * LD + c] -= s[i * LD + j] * s[c * LD + j];
    }
    __syncthreads();
  }
  const int b = bad;
  if (b == 0)
    for (int e = threadIdx.x; e < nb * nb; e += NT) {
      const int i = e / nb, j = e % nb;
      if (j <= i) A[(j0 + i) * ld + j0 + j] = s[i * LD + j];
    }
  return b;
}

__global__ void __launch_bounds__(NT) chol_fused_kernel(CholArgs a) {
  extern __shared__ double smem[];
  cg::grid_group grid = cg::this_grid();
  double* A = a.A;
  const int dim = a.dim;
  const long long ld = a.ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gwarp = blockIdx.x * (NT / 32) + warp, nwarps = gridDim.x * (NT / 32);

  // ---- lam = max abs row sum of the original matrix (one warp per row)
  for (int row = gwarp; row < dim; row += nwarps) {
    double s = 0.0;
    for (int j = lane; j < dim; j += 32) s += fabs(A[row * ld + j]);
    s = warp_sum(s);
    if (lane == 0) atomicMax((unsigned long long*)a.lam, (unsigned long long)__double_as_longlong(s));
  }
  grid.sync();

  // ---- blocked right-looking Cholesky
  for (int j0 = 0; j0 < dim; j0 += NB) {
    const int nb = min(NB, dim - j0);
    if (blockIdx.x == 0) {
      const int b = factor_diag(A, ld, j0, nb, smem);
      if (threadIdx.x == 0 && b != 0) *a.info = b;
    }
    grid.sync();
    if (__ldcg(a.info) != 0) return;  // uniform: every CTA reads the same flag
    const int rest = dim - j0 - nb;
    if (rest <= 0) break;
    // panel solve: L21 = A21 L11^-T, one thread per row, L11 staged in shared memory
    {
      constexpr int LD = NB + 1;
      double* L = smem;
      for (int e = threadIdx.x; e < nb * nb; e += NT) {
        const int i = e / nb, j = e % nb;
        L[i * LD + j] = (j <= i) ? __ldcg(A + (j0 + i) * ld + j0 + j) : 0.0;
      }
      __syncthreads();
      for (int row = j0 + nb + blockIdx.x * NT + threadIdx.x; row < dim; row += gridDim.x * NT) {
        double x[NB];
        double* ar = A + row * ld + j0;
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
  }

  // ---- triangular solves on x (= b on entry), block by block
  double* x = a.x;
  __shared__ double xb[NB];
  // forward: L y = b
  for (int j0 = 0; j0 < dim; j0 += NB) {
    const int nb = min(NB, dim - j0);
    if (blockIdx.x == 0) {
      if (warp == 0) {
        // two lanes-halves: rows j0+lane and j0+32+lane
        double v0 = lane < nb ? __ldcg(x + j0 + lane) : 0.0;
        double v1 = lane + 32 < nb ? __ldcg(x + j0 + 32 + lane) : 0.0;
        for (int j = 0; j < nb; ++j) {
          const double src = j < 32 ? __shfl_sync(0xffffffffu, v0, j) : __shfl_sync(0xffffffffu, v1, j - 32);
          const double xj = src / __ldcg(A + (long long)(j0 + j) * ld + j0 + j);
          const int r0 = lane, r1 = lane + 32;
          if (r0 == j) v0 = xj;
          else if (r0 > j && r0 < nb) v0 -= __ldcg(A + (long long)(j0 + r0) * ld + j0 + j) * xj;
          if (r1 == j) v1 = xj;
          else if (r1 > j && r1 < nb) v1 -= __ldcg(A + (long long)(j0 + r1) * ld + j0 + j) * xj;
        }
        if (lane < nb) x[j0 + lane] = v0;
        if (lane + 32 < nb) x[j0 + 32 + lane] = v1;
      }
    }
    grid.sync();
    for (int e = threadIdx.x; e < nb; e += NT) xb[e] = __ldcg(x + j0 + e);
    __syncthreads();
    for (int row = j0 + nb + gwarp; row < dim; row += nwarps) {  // one warp per row
      double s = 0.0;
      for (int j = lane; j < nb; j += 32) s += A[(long long)row * ld + j0 + j] * xb[j];
      s = warp_sum(s);
      if (lane == 0) x[row] -= s;
    }
    __syncthreads();
    grid.sync();
  }
  // backward: L^T x = y
  for (int j1 = dim; j1 > 0; j1 -= NB) {
    const int j0 = max(0, j1 - NB), nb = j1 - j0;
    if (blockIdx.x == 0) {
      if (warp == 0) {
        double v0 = lane < nb ? __ldcg(x + j0 + lane) : 0.0;
        double v1 = lane + 32 < nb ? __ldcg(x + j0 + 32 + lane) : 0.0;
        for (int j = nb - 1; j >= 0; --j) {
          const double src = j < 32 ? __shfl_sync(0xffffffffu, v0, j) : __shfl_sync(0xffffffffu, v1, j - 32);
          const double xj = src / __ldcg(A + (long long)(j0 + j) * ld + j0 + j);
          const int r0 = lane, r1 = lane + 32;
          // L^T[r, j] = L[j, r] for r < j
          if (r0 == j) v0 = xj;
          else if (r0 < j) v0 -= __ldcg(A + (long long)(j0 + j) * ld + j0 + r0) * xj;
          if (r1 == j) v1 = xj;
          else if (r1 < j) v1 -= __ldcg(A + (long long)(j0 + j) * ld + j0 + r1) * xj;
        }
        if (lane < nb) x[j0 + lane] = v0;
        if (lane + 32 < nb) x[j0 + 32 + lane] = v1;
      }
    }
    grid.sync();
    for (int e = threadIdx.x; e < nb; e += NT) xb[e] = __ldcg(x + j0 + e);
    __syncthreads();
    // x[i] -= sum_j L[j0+j, i] x[j0+j] for i < j0 (coalesced over i)
    for (int i = blockIdx.x * NT + threadIdx.x; i < j0; i += gridDim.x * NT) {
      double s = 0.0;
      for (int j = 0; j < nb; ++j) s += A[(long long)(j0 + j) * ld + i] * xb[j];
      x[i] -= s;
    }
    __syncthreads();
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

void chol_fused_launch(const CholArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  QTT_CUDA(cudaLaunchCooperativeKernel((void*)chol_fused_kernel, dim3(grid), dim3(NT), args, CF::SMEM, s));
  QTT_CHECK_LAUNCH();
}

}  // namespace qtt
