// Persistent, cooperative Jacobi-PCG for one AMEn local system (amen.py:192-214):
// every iteration -- the three-GEMM local matvec (amen.py:134-137) on the DMMA tile
// engine, the split-K reduction, the dot products and the vector updates -- runs
// inside ONE kernel launch, phases separated by grid-wide barriers, so nothing
// leaves HBM/L2 between iterations and there is no per-iteration launch or host
// round trip (north_star item c).  Reductions are fixed-order (deterministic) and
// every CTA evaluates the same scalar recurrence, so all CTAs agree on the SciPy
// stopping rule  ||r|| < rtol*||b||  checked before each step.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "cg_fused.cuh"
#include "dmma_tile.cuh"
#include "gemm.cuh"

namespace cg = cooperative_groups;

namespace qtt {
namespace {

using CF = tile::Cfg<64, 64, 16, 2, 4, 3>;  // 256 threads, warp tile 32x16
constexpr int NT = CF::NT;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sums of two values, broadcast (red: >= 20 doubles of shared memory)
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) { red[warp] = a; red[8 + warp] = b; }
  __syncthreads();
  if (warp == 0) {
    double x = lane < NT / 32 ? red[lane] : 0.0, y = lane < NT / 32 ? red[8 + lane] : 0.0;
    x = warp_sum(x);
    y = warp_sum(y);
    if (lane == 0) { red[16] = x; red[17] = y; }
  }
  __syncthreads();
  a = red[16];
  b = red[17];
  __syncthreads();
}

// Sum the per-CTA partials part[2*i + {0,1}] in a fixed order (identical in every CTA).
__device__ __forceinline__ void grid_sum2(const double* part, int nparts, double& a, double& b, double* red) {
  a = 0.0;
  b = 0.0;
  for (int i = threadIdx.x; i < nparts; i += NT) {
    a += __ldcg(part + 2 * i);
    b += __ldcg(part + 2 * i + 1);
  }
  block_sum2(a, b, red);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One GEMM phase: every CTA takes work items blockIdx.x, +gridDim.x, ...
// C[b][r*c_rs + c] = sum_k op(A_b)(r,k) op(B_b)(k,c)   (split-K when splits > 1:
// item writes its partial into C + s*split_stride instead)
template <class T>
__device__ __noinline__ void phase_gemm(const tile::Operands& o0, long long a_bs, long long b_bs, int batch, double* C,
                           long long c_rs, long long c_bs, int splits, int kt_per, long long split_stride,
                           double* smem) {
  const int tm = (o0.M + T::BM - 1) / T::BM, tn = (o0.N + T::BN - 1) / T::BN;
  const int ktiles = (o0.K + T::BK - 1) / T::BK;
  const long long per_batch = (long long)tm * tn * splits;
  const long long items = per_batch * batch;
  // this CTA's items: blockIdx.x, +gridDim.x, ... streamed through one cp.async ring
  const int mine = items > blockIdx.x ? (int)((items - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  auto decode = [&](int i, int& b, int& s) {
    const long long it = blockIdx.x + (long long)i * gridDim.x;
    b = (int)(it / per_batch);
    long long rem = it % per_batch;
    s = (int)(rem % splits);
    rem /= splits;
    return rem;
  };
  auto get = [&](int i) {
    int b, s;
    const long long rem = decode(i, b, s);
    tile::TileItem t;
    t.o = o0;
    t.o.A += b * a_bs;
    t.o.B += b * b_bs;
    t.m0 = (int)(rem / tn) * T::BM;
    t.n0 = (int)(rem % tn) * T::BN;
    t.kb = s * kt_per;
    t.ke = min(ktiles, t.kb + kt_per);
    return t;
  };
  int cur = 0;
  auto epi = [&](const tile::TileItem& t, const double (&acc)[T::MI][T::NI][2]) {
    int b, s;
    decode(cur++, b, s);
    double* Cb = C + b * c_bs + s * split_stride;
    tile::for_each_acc<T>(t.m0, t.n0, t.o.M, t.o.N, acc,
                          [&](int r, int c, double v) { Cb[(long long)r * c_rs + c] = v; });
  };
  tile::mma_stream<T>(mine, get, epi, smem);
}

// Tile shapes selectable per phase (CGFusedArgs::tileA / tile3): the local ranks
// (~96-112 at the C3 rank cap) make 64x64 tiles 60-80% full, so wider N tiles
// that cover the whole rank in one tile are offered too.
using T64x64 = CF;
using T64x112 = tile::Cfg<64, 112, 16, 4, 2, 3>;  // warp tile 16x56
using T32x112 = tile::Cfg<32, 112, 16, 4, 2, 3>;  // warp tile 8x56
using T64x96 = tile::Cfg<64, 96, 16, 4, 2, 3>;    // warp tile 16x48
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t SMEM_MAX = cmax(cmax(T64x64::SMEM, T64x112::SMEM), cmax(T32x112::SMEM, T64x96::SMEM));

template <class... Args>
__device__ void phase_gemm_sel(int sel, Args... args) {
  switch (sel) {
    case 1: phase_gemm<T64x112>(args...); break;
    case 2: phase_gemm<T32x112>(args...); break;
    case 3: phase_gemm<T64x96>(args...); break;
    default: phase_gemm<T64x64>(args...); break;
  }
}

// q = A v  for the local operator, leaves q = sum of the split-K partials of step 3
// unreduced in a.part3; returns after a grid barrier.
__device__ __forceinline__ void phase_mark(const CGFusedArgs& a, int ph, unsigned long long& t) {
  if (a.phase_ns != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long now = gtimer();
    a.phase_ns[ph] += now - t;
    t = now;
  }
}

__device__ void matvec_phases(const CGFusedArgs& a, const double* v, double* smem, cg::grid_group& grid,
                              unsigned long long& tp) {
  if (a.Bop != nullptr) {
    // steps 1+2 composed, one GEMM over all X: t2[(X,m,b),V] = Bop[(X,m,b),(U,n)] @ v[(U,n),V]
    tile::Operands oc{a.Bop, (long long)a.lk * a.n, 1, v, a.rk, 1, a.lb * a.m * a.R1, a.rk, a.lk * a.n};
    phase_gemm_sel(a.tileA, oc, 0LL, 0LL, 1, a.t2, (long long)a.rk, 0LL, 1, (oc.K + 15) / 16, 0LL, smem);
    grid.sync();
    phase_mark(a, 1, tp);
  } else {
    // step 1: t1[(X,a),(n,V)] = phil[(X,a),U] @ v[U,(n,V)]
    tile::Operands o1{a.phil, a.lk, 1, v, (long long)a.n * a.rk, 1, a.lb * a.lo, a.n * a.rk, a.lk};
    phase_gemm_sel(0, o1, 0LL, 0LL, 1, a.t1, (long long)a.n * a.rk, 0LL, 1, (o1.K + 15) / 16, 0LL, smem);
    grid.sync();
    phase_mark(a, 0, tp);
    // step 2: per X: t2[X][(m,b),V] = Ap[(m,b),(a,n)] @ t1[X][(a,n),V]
    tile::Operands o2{a.Ap, (long long)a.lo * a.n, 1, a.t1, a.rk, 1, a.m * a.R1, a.rk, a.lo * a.n};
    phase_gemm_sel(a.tileA, o2, 0LL, (long long)a.lo * a.n * a.rk, a.lb, a.t2, (long long)a.rk,
                   (long long)a.m * a.R1 * a.rk, 1, (o2.K + 15) / 16, 0LL, smem);
    grid.sync();
    phase_mark(a, 1, tp);
  }
  // step 3 (split-K): part3[s][(X,m),Y] = t2[(X,m),(b,V)] @ phir[Y,(b,V)]^T
  tile::Operands o3{a.t2, (long long)a.R1 * a.rk, 1, a.phir, 1, (long long)a.R1 * a.rk, a.lb * a.m, a.rb,
                    a.R1 * a.rk};
  phase_gemm_sel(a.tile3, o3, 0LL, 0LL, 1, a.part3, (long long)a.rb, 0LL, a.S3, a.kt_per3,
                 (long long)a.lb * a.m * a.rb, smem);
  grid.sync();
  phase_mark(a, 2, tp);
}

__device__ __forceinline__ double reduce_q(const CGFusedArgs& a, long long e) {
  double s = 0.0;
  const long long stride = a.dim;
  for (int k = 0; k < a.S3; ++k) s += __ldcg(a.part3 + k * stride + e);
  return s;
}

__global__ void __launch_bounds__(NT, 2) cg_fused_kernel(CGFusedArgs a) {
  extern __shared__ double smem[];
  __shared__ double red[24];
  cg::grid_group grid = cg::this_grid();
  const long long n = a.dim;
  // contiguous slice of the vectors owned by this CTA
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long e0 = blockIdx.x * per, e1 = min(n, e0 + per);
  unsigned long long mv_ns = 0, t0 = 0, tp = gtimer();
  const bool timer = (blockIdx.x == 0 && threadIdx.x == 0);

  // ---- r = b - A x0 (only when x0 has a nonzero entry, as scipy's `x.any()`)
  if (a.xany) {
    if (timer) t0 = gtimer();
    matvec_phases(a, a.x, smem, grid, tp);
    if (timer) mv_ns += gtimer() - t0;
  }
  double rr = 0.0, rz = 0.0;
  for (long long e = e0 + threadIdx.x; e < e1; e += NT) {
    const double ri = a.xany ? __ldcg(a.b + e) - reduce_q(a, e) : __ldcg(a.b + e);
    const double zi = ri * a.invd[e];
    a.r[e] = ri;
    a.z[e] = zi;
    a.p[e] = zi;
    rr += ri * ri;
    rz += ri * zi;
  }
  block_sum2(rr, rz, red);
  if (threadIdx.x == 0) { a.red[2 * blockIdx.x] = rr; a.red[2 * blockIdx.x + 1] = rz; }
  grid.sync();
  grid_sum2(a.red, gridDim.x, rr, rz, red);
  double rho = rz, rnorm = sqrt(rr);
  int it = 0;
  // p.q partials go to a second buffer, so no extra barrier is needed before reuse
  double* red_pq = a.red + 2 * gridDim.x;

  while (!(rnorm < a.atol) && it < a.maxiter) {
    // ---- q = A p
    if (timer) t0 = gtimer();
    matvec_phases(a, a.p, smem, grid, tp);
    // ---- reduce q, p.q
    double pq = 0.0, dummy = 0.0;
    for (long long e = e0 + threadIdx.x; e < e1; e += NT) {
      const double qi = reduce_q(a, e);
      a.q[e] = qi;
      pq += __ldcg(a.p + e) * qi;
    }
    block_sum2(pq, dummy, red);
    if (threadIdx.x == 0) { red_pq[2 * blockIdx.x] = pq; red_pq[2 * blockIdx.x + 1] = 0.0; }
    grid.sync();
    phase_mark(a, 3, tp);
    if (timer) mv_ns += gtimer() - t0;
    grid_sum2(red_pq, gridDim.x, pq, dummy, red);
    const double alpha = rho / pq;
    // ---- x += alpha p; r -= alpha q; z = M^-1 r; rr, rz
    rr = 0.0;
    rz = 0.0;
    for (long long e = e0 + threadIdx.x; e < e1; e += NT) {
      const double pi = __ldcg(a.p + e);
      a.x[e] += alpha * pi;
      const double ri = a.r[e] - alpha * a.q[e];
      a.r[e] = ri;
      const double zi = ri * a.invd[e];
      a.z[e] = zi;
      rr += ri * ri;
      rz += ri * zi;
    }
    block_sum2(rr, rz, red);
    if (threadIdx.x == 0) { a.red[2 * blockIdx.x] = rr; a.red[2 * blockIdx.x + 1] = rz; }
    grid.sync();
    phase_mark(a, 4, tp);
    grid_sum2(a.red, gridDim.x, rr, rz, red);
    ++it;
    rnorm = sqrt(rr);
    if (rnorm < a.atol || it >= a.maxiter) break;
    const double beta = rz / rho;
    rho = rz;
    for (long long e = e0 + threadIdx.x; e < e1; e += NT) a.p[e] = a.z[e] + beta * a.p[e];
    grid.sync();
    phase_mark(a, 5, tp);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.out_iters = it;
    *a.out_rnorm = rnorm;
    *a.out_mv_ns += mv_ns;
  }
}

}  // namespace

int cg_fused_grid(int device) {
  static PerDevice<int> cache(-1);
  int& cached = cache.at(device);
  if (cached > 0) return cached;
  QTT_CUDA(cudaFuncSetAttribute(cg_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_MAX));
  int per_sm = 0, sms = 0;
  QTT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_fused_kernel, NT, SMEM_MAX));
  QTT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  cached = std::max(1, std::min(per_sm, 2)) * sms;
  return cached;
}

int tile_bm(int sel) { return sel == 2 ? 32 : 64; }
int tile_bn(int sel) { return sel == 1 || sel == 2 ? 112 : (sel == 3 ? 96 : 64); }

// Tile shape for an N-wide phase: one tile spanning N when N is just above a
// multiple of 64 (rank ~96-112), else 64x64.  QTT_CG_TILE_A / _3 force a shape.
int pick_tile(int N, const char* env) {
  if (const char* e = std::getenv(env)) return std::atoi(e);
  if (N > 64 && N <= 96) return 3;
  if (N > 96 && N <= 112) return 1;
  return 0;
}

void cg_fused_plan(int lb, int m, int rb, int R1, int rk, int grid, int& S3, int& kt_per3, int& tileA,
                   int& tile3) {
  tileA = pick_tile(rk, "QTT_CG_TILE_A");
  tile3 = pick_tile(rb, "QTT_CG_TILE_3");
  const int M3 = lb * m, N3 = rb, K3 = R1 * rk;
  const int tiles = cdiv(M3, tile_bm(tile3)) * cdiv(N3, tile_bn(tile3));
  const int ktiles = cdiv(K3, 16);
  // as many K slices as fit in one wave of the grid (no second round of tiles)
  static const int cap = std::getenv("QTT_CG_S3CAP") ? std::atoi(std::getenv("QTT_CG_S3CAP")) : 1 << 20;
  int want = std::max(1, std::min({grid / std::max(1, tiles), std::max(1, ktiles / 4), cap}));
  kt_per3 = cdiv(ktiles, want);
  S3 = cdiv(ktiles, kt_per3);
}

double cg_fused_flops(int lb, int lo, int lk, int m, int n, int R1, int rb, int rk, bool composed) {
  const double s3 = 2.0 * lb * m * rb * (double)R1 * rk;
  if (composed) return 2.0 * lb * (double)m * R1 * lk * n * rk + s3;
  return 2.0 * lb * (double)lo * lk * n * rk + 2.0 * lb * (double)m * R1 * lo * n * rk + s3;
}

void cg_fused_build_bop(const double* phil, int lb, int lo, int lk, const double* Ap, int m, int n, int R1,
                        double* Bop, cudaStream_t s) {
  // batched over (X, n'):  Bop[X][(m,b)][U][n'] = sum_a Ap[(m,b)][a][n'] phil[X][a][U]
  GemmArgs g;
  g.M = m * R1; g.N = lk; g.K = lo;
  g.A = Ap; g.a_rs = (long long)lo * n; g.a_cs = n; g.a_bs1 = 0; g.a_bs2 = 1;
  g.B = phil; g.b_rs = lk; g.b_cs = 1; g.b_bs1 = (long long)lo * lk; g.b_bs2 = 0;
  g.C = Bop; g.c_rs = (long long)lk * n; g.c_cs = n; g.c_bs1 = (long long)m * R1 * lk * n; g.c_bs2 = 1;
  g.batch1 = lb; g.batch2 = n;
  gemm(g, s, nullptr, 0);
}

void cg_fused_launch(const CGFusedArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  QTT_CUDA(cudaLaunchCooperativeKernel((void*)cg_fused_kernel, dim3(grid), dim3(NT), args, SMEM_MAX, s));
  QTT_CHECK_LAUNCH();
}

}  // namespace qtt
