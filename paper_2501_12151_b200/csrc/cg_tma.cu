// Persistent cooperative Jacobi-PCG (amen.py:192-214, SciPy cg recurrence) whose
// local matvec runs on the TMA tile engine (tma_tile.cuh).  Per iteration:
//   phase 1  t2[(X,m,b),V] = sum_(U,n) Bop[(X,m,b),(U,n)] p^T[V,(U,n)]
//            (Bop = left environment composed with the operator core, built once per
//            solve; one GEMM over all X, balanced over the grid by stream-K: every CTA
//            takes an equal run of k-tiles, split tiles are finished in a fixed order)
//   phase 2  q^T[Y,(X,m)] = sum_(b,V) phir[Y,(b,V)] t2[(X,m),(b,V)]   (split-K)
//   then the split-K reduction + p.q, the x/r/z update + r.r, r.z, and p = z + beta p,
// phases separated by grid barriers, everything resident in L2/HBM between them.
// Vectors are stored transposed ([V][U][n]) so both GEMMs read K-contiguous rows.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "cg_tma.cuh"
#include "tma_tile.cuh"

namespace cg = cooperative_groups;

namespace qtt {
namespace {

constexpr int NT = 256;
using C64 = tma::Cfg<64, 64, 2, 4, 4>;       // warp tile 32x16
using C64x112 = tma::Cfg<64, 112, 4, 2, 4>;  // warp tile 16x56
using C112x64 = tma::Cfg<112, 64, 2, 4, 4>;  // warp tile 56x16
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t SMEM = cmax(C64::SMEM, cmax(C64x112::SMEM, C112x64::SMEM));
constexpr long long TILE_DOUBLES = 64 * 112;  // largest BM*BN (stream-K partial slot)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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

__device__ __forceinline__ void phase_mark(const CGTmaArgs& a, int ph, unsigned long long& t) {
  if (a.phase_ns != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long now = gtimer();
    a.phase_ns[ph] += now - t;
    t = now;
  }
}

// generic-proxy global writes -> later TMA (async-proxy) reads, across the grid barrier
__device__ __forceinline__ void fence_proxy_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- phase 1 (stream-K): t2 <- Bop . v^T
template <class T>
__device__ __noinline__ void phase1(const CGTmaArgs& a, const CUtensorMap* mv, tma::Ring& ring, unsigned epoch) {
  const int M = a.lb * a.m * a.R1, N = a.rk, K = a.lk * a.n;
  const int tn = (N + T::BN - 1) / T::BN;
  const int tm = (M + T::BM - 1) / T::BM;
  const int KT = (K + 15) / 16;
  const long long U = (long long)tm * tn * KT;
  const int G = gridDim.x, c = blockIdx.x;
  const long long u0 = U * c / G, u1 = U * (c + 1) / G;
  if (u0 >= u1) return;
  const int t_first = (int)(u0 / KT), t_last = (int)((u1 - 1) / KT);
  const CUtensorMap* mb = &a.map_bop;
  auto get = [&](int i) {
    tma::Item it;
    it.ma = mb;
    it.mb = mv;
    const int t = t_first + i;
    it.m0 = (t / tn) * T::BM;
    it.n0 = (t % tn) * T::BN;
    it.kb = (int)max(0LL, u0 - (long long)t * KT);
    it.ke = (int)min((long long)KT, u1 - (long long)t * KT);
    return it;
  };
  const int R1 = a.R1, rk = a.rk;
  const long long K3p = a.K3p;
  double* t2 = a.t2;
  auto store = [&](const tma::Item& it, const double (&acc)[T::MI][T::NI][2]) {
    tma::for_each<T>(it.m0, it.n0, M, N, acc, [&](int r, int col, double v) {
      const int xm = r / R1, bb = r - xm * R1;
      t2[xm * K3p + (long long)bb * rk + col] = v;
    });
  };
  auto epi = [&](const tma::Item& it, const double (&acc)[T::MI][T::NI][2]) {
    if (it.kb == 0 && it.ke == KT) {
      store(it, acc);
      return;
    }
    if (it.kb > 0) {  // contributor: publish the partial tile, fragment order (coalesced)
      double* w = a.sk_ws + (long long)c * TILE_DOUBLES;
      int e = 0;
#pragma unroll
      for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) w[(e++) * NT + threadIdx.x] = acc[i][j][h];
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release(a.sk_flags + c, epoch);
      return;
    }
    // finisher (owns k-tile 0): add the later CTAs' partials in CTA order (deterministic)
    auto& sum = const_cast<double(&)[T::MI][T::NI][2]>(acc);  // the stream's own accumulator
    const long long t = (long long)(it.m0 / T::BM) * tn + it.n0 / T::BN;
    const long long tile_end = (t + 1) * KT;
    for (int c2 = c + 1; c2 < G; ++c2) {
      const long long s2 = U * c2 / G, e2 = U * (c2 + 1) / G;
      if (s2 >= tile_end) break;
      if (s2 >= e2) continue;
      if (threadIdx.x == 0)
        while (ld_acquire(a.sk_flags + c2) < epoch) {
        }
      __syncthreads();
      const double* w = a.sk_ws + (long long)c2 * TILE_DOUBLES;
      int e = 0;
#pragma unroll
      for (int i = 0; i < T::MI; ++i)
#pragma unroll
        for (int j = 0; j < T::NI; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) sum[i][j][h] += __ldcg(w + (e++) * NT + threadIdx.x);
    }
    store(it, sum);
  };
  tma::stream<T>(ring, t_last - t_first + 1, get, epi);
}

// ---- phase 2 (split-K): part3[s][Y][(X,m)] = phir[Y, slice s] . t2[(X,m), slice s]
template <class T>
__device__ __noinline__ void phase2(const CGTmaArgs& a, tma::Ring& ring) {
  const int M = a.rb, N = a.lb * a.m, K = a.R1 * a.rk;
  const int tm = (M + T::BM - 1) / T::BM, tn = (N + T::BN - 1) / T::BN;
  const int KT = (K + 15) / 16;
  const int S = a.S3, ktp = a.kt_per3;
  const int items = tm * tn * S;
  const int mine = items > (int)blockIdx.x ? (items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto get = [&](int i) {
    const int it = blockIdx.x + i * gridDim.x;
    const int s = it % S, tile = it / S;
    tma::Item r;
    r.ma = &a.map_phir;
    r.mb = &a.map_t2;
    r.m0 = (tile / tn) * T::BM;
    r.n0 = (tile % tn) * T::BN;
    r.kb = s * ktp;
    r.ke = min(KT, r.kb + ktp);
    return r;
  };
  const long long dim = a.dim;
  double* part3 = a.part3;
  auto epi = [&](const tma::Item& it, const double (&acc)[T::MI][T::NI][2]) {
    double* P = part3 + (long long)(it.kb / ktp) * dim;
    tma::for_each<T>(it.m0, it.n0, M, N, acc, [&](int r, int col, double v) { P[(long long)r * N + col] = v; });
  };
  tma::stream<T>(ring, mine, get, epi);
}

__device__ void matvec(const CGTmaArgs& a, const CUtensorMap* mv, tma::Ring& ring, unsigned& epoch,
                       cg::grid_group& grid, unsigned long long& tp) {
  ++epoch;
  const unsigned long long ts = a.cta_ns != nullptr ? gtimer() : 0;
  if (a.cfg1 == 1)
    phase1<C64x112>(a, mv, ring, epoch);
  else
    phase1<C64>(a, mv, ring, epoch);
  if (a.cta_ns != nullptr && threadIdx.x == 0) a.cta_ns[blockIdx.x] += gtimer() - ts;
  const unsigned long long ts2 = a.cta_ns != nullptr ? gtimer() : 0;
  fence_proxy_global();
  grid.sync();
  phase_mark(a, 1, tp);
  if (a.cfg2 == 1)
    phase2<C112x64>(a, ring);
  else
    phase2<C64>(a, ring);
  if (a.cta_ns != nullptr && threadIdx.x == 0) a.cta_ns[gridDim.x + blockIdx.x] += gtimer() - ts2;
  grid.sync();
  phase_mark(a, 2, tp);
}

// Split-K reduction of this CTA's slice [e0, e1): KS consecutive lanes (a power of
// two) share one element and take its partials k = g, g+KS, ...; their sums are
// combined by a fixed xor tree, so the result is deterministic.  f(e, q) is called
// by the group's lane 0.
template <class F>
__device__ __forceinline__ void reduce_slice(const CGTmaArgs& a, long long e0, long long e1, F&& f) {
  const int cnt = (int)(e1 - e0);
  if (cnt <= 0) return;
  const int S = a.S3;
  int KS = 1;
  while (KS * 2 <= S && KS * 2 <= 32 && KS * 2 * cnt <= NT) KS *= 2;
  const int g = threadIdx.x & (KS - 1);
  const long long dim = a.dim;
  const double* part = a.part3;
  // every lane of a warp runs the same number of element rounds (shuffles below)
  const int rounds = (cnt + NT / KS - 1) / (NT / KS);
  for (int rd = 0; rd < rounds; ++rd) {
    const int el = rd * (NT / KS) + (int)threadIdx.x / KS;
    const long long e = e0 + el;
    double s = 0.0;
    if (el < cnt) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int k = g;
      for (; k + 3 * KS < S; k += 4 * KS) {
        s0 += __ldcg(part + k * dim + e);
        s1 += __ldcg(part + (k + KS) * dim + e);
        s2 += __ldcg(part + (k + 2 * KS) * dim + e);
        s3 += __ldcg(part + (k + 3 * KS) * dim + e);
      }
      for (; k < S; k += KS) s0 += __ldcg(part + k * dim + e);
      s = (s0 + s1) + (s2 + s3);
    }
    for (int o = 1; o < KS; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (el < cnt && g == 0) f(e, s);
  }
}

__global__ void __launch_bounds__(NT, 2) cg_tma_kernel(const __grid_constant__ CGTmaArgs a) {
  extern __shared__ unsigned char smem_raw[];
  __shared__ double red[24];
  cg::grid_group grid = cg::this_grid();
  const long long n = a.dim;
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long e0 = blockIdx.x * per, e1 = min(n, e0 + per);
  unsigned long long mv_ns = 0, t0 = 0, tp = gtimer();
  const bool timer = (blockIdx.x == 0 && threadIdx.x == 0);
  tma::Ring ring = tma::ring_init<4>(smem_raw);
  if (threadIdx.x == 0) {
    a.sk_flags[blockIdx.x] = 0u;
    tma::prefetch_map(&a.map_bop);
    tma::prefetch_map(&a.map_p);
    tma::prefetch_map(&a.map_phir);
    tma::prefetch_map(&a.map_t2);
  }
  unsigned epoch = 0;
  if (a.cta_ns != nullptr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.cta_ns[2 * gridDim.x + blockIdx.x] = smid;
  }
  grid.sync();

  // ---- r = b - A x0 (only when x0 has a nonzero entry, as scipy's `x.any()`)
  if (a.xany) {
    if (timer) t0 = gtimer();
    matvec(a, &a.map_x, ring, epoch, grid, tp);
    if (timer) mv_ns += gtimer() - t0;
  }
  double rr = 0.0, rz = 0.0;
  auto init_r = [&](long long e, double ax) {
    const double ri = __ldcg(a.b + e) - ax;
    const double zi = ri * a.invd[e];
    a.r[e] = ri;
    a.z[e] = zi;
    a.p[e] = zi;
    rr += ri * ri;
    rz += ri * zi;
  };
  if (a.xany)
    reduce_slice(a, e0, e1, init_r);
  else
    for (long long e = e0 + threadIdx.x; e < e1; e += NT) init_r(e, 0.0);
  fence_proxy_global();
  block_sum2(rr, rz, red);
  if (threadIdx.x == 0) { a.red[2 * blockIdx.x] = rr; a.red[2 * blockIdx.x + 1] = rz; }
  grid.sync();
  grid_sum2(a.red, gridDim.x, rr, rz, red);
  double rho = rz, rnorm = sqrt(rr);
  int it = 0;
  double* red_pq = a.red + 2 * gridDim.x;

  while (!(rnorm < a.atol) && it < a.maxiter) {
    if (timer) t0 = gtimer();
    matvec(a, &a.map_p, ring, epoch, grid, tp);
    double pq = 0.0, dummy = 0.0;
    reduce_slice(a, e0, e1, [&](long long e, double qi) {
      a.q[e] = qi;
      pq += __ldcg(a.p + e) * qi;
    });
    block_sum2(pq, dummy, red);
    if (threadIdx.x == 0) { red_pq[2 * blockIdx.x] = pq; red_pq[2 * blockIdx.x + 1] = 0.0; }
    grid.sync();
    phase_mark(a, 3, tp);
    if (timer) mv_ns += gtimer() - t0;
    grid_sum2(red_pq, gridDim.x, pq, dummy, red);
    const double alpha = rho / pq;
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
    fence_proxy_global();
    grid.sync();
    phase_mark(a, 5, tp);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.out_iters = it;
    *a.out_rnorm = rnorm;
    *a.out_mv_ns += mv_ns;
  }
}

__global__ void transpose_kernel(const double* __restrict__ in, double* __restrict__ out, long long rows,
                                 long long cols) {
  __shared__ double tile[32][33];
  const long long r0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const long long r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const long long c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
  }
}

}  // namespace

bool cg_tma_supported(int lk, int n) { return ((long long)lk * n) % 2 == 0; }

int cg_tma_grid(int device) {
  static int cached = -1;
  if (cached > 0) return cached;
  QTT_CUDA(cudaFuncSetAttribute(cg_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  int per_sm = 0, sms = 0;
  QTT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_tma_kernel, NT, SMEM));
  QTT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  static const int want = std::getenv("QTT_TMA_PER_SM") ? std::atoi(std::getenv("QTT_TMA_PER_SM")) : 1;
  cached = std::max(1, std::min(per_sm, want)) * sms;
  return cached;
}

long long cg_tma_tile_doubles() { return TILE_DOUBLES; }

CGTmaPlan cg_tma_plan(int lb, int m, int R1, int lk, int n, int rb, int rk, int grid) {
  (void)lk;
  (void)n;
  CGTmaPlan p{};
  static const int f1 = std::getenv("QTT_TMA_CFG1") ? std::atoi(std::getenv("QTT_TMA_CFG1")) : -1;
  static const int f2 = std::getenv("QTT_TMA_CFG2") ? std::atoi(std::getenv("QTT_TMA_CFG2")) : -1;
  p.cfg1 = f1 >= 0 ? f1 : (rk > 64 ? 1 : 0);
  p.cfg2 = f2 >= 0 ? f2 : (rb > 64 ? 1 : 0);
  p.box1_a = 64;
  p.box1_b = p.cfg1 == 1 ? 112 : 64;
  p.box2_a = p.cfg2 == 1 ? 112 : 64;
  p.box2_b = 64;
  const int M3 = rb, N3 = lb * m, K3 = R1 * rk;
  const int tiles = cdiv(M3, p.box2_a) * cdiv(N3, p.box2_b);
  const int ktiles = cdiv(K3, 16);
  int want = std::max(1, std::min(grid / std::max(1, tiles), std::max(1, ktiles / 4)));
  p.kt_per3 = cdiv(ktiles, want);
  p.S3 = cdiv(ktiles, p.kt_per3);
  return p;
}

void cg_tma_launch(const CGTmaArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  QTT_CUDA(cudaLaunchCooperativeKernel((void*)cg_tma_kernel, dim3(grid), dim3(NT), args, SMEM, s));
  QTT_CHECK_LAUNCH();
}

void transpose_2d(const double* in, double* out, long long rows, long long cols, cudaStream_t s) {
  dim3 g((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32));
  transpose_kernel<<<g, dim3(32, 8), 0, s>>>(in, out, rows, cols);
  QTT_CHECK_LAUNCH();
}

}  // namespace qtt
