// Persistent cooperative Jacobi-PCG (amen.py:192-214, SciPy cg recurrence) whose
// local matvec runs on the TMA tile engine (tma_tile.cuh).  Per iteration:
//   phase 1  t2[(X,m,b),V] = sum_(U,n) Bop[(X,m,b),(U,n)] p^T[V,(U,n)]
//            (Bop = left environment composed with the operator core, built once per
//            solve; one GEMM over all X, every CTA an exact 1/148 share of the output
//            fragments, dealt evenly to its warps -- tma_fb.cuh)
//   phase 2  q^T[Y,(X,m)] = sum_(b,V) phir[Y,(b,V)] t2[(X,m),(b,V)]   (split-K)
//   then the split-K reduction + p.q, the x/r/z update + r.r, r.z, and p = z + beta p,
// phases separated by grid barriers, everything resident in L2/HBM between them.
// Vectors are stored transposed ([V][U][n]) so both GEMMs read K-contiguous rows.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "cg_tma.cuh"
#include "tma_fb.cuh"

namespace cg = cooperative_groups;

namespace qtt {
namespace {

constexpr int NW = 12;        // 12 warps (3 per scheduler: the register file holds 3 x 168 per scheduler)
constexpr int NTC = NW * 32;  // one CTA per SM
constexpr int NT = NTC;
static_assert(NW == tmafb::NWARP, "fragment dealing uses every warp");

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sums of two values, broadcast (red: >= 2*NW + 2 doubles of shared memory)
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0 && warp < NW) { red[warp] = a; red[NW + warp] = b; }
  __syncthreads();
  if (warp == 0) {
    double x = lane < NW ? red[lane] : 0.0, y = lane < NW ? red[NW + lane] : 0.0;
    x = warp_sum(x);
    y = warp_sum(y);
    if (lane == 0) { red[2 * NW] = x; red[2 * NW + 1] = y; }
  }
  __syncthreads();
  a = red[2 * NW];
  b = red[2 * NW + 1];
  __syncthreads();
}

// Sum of the per-CTA partial pairs (one load per thread, then a block reduction: measured
// faster than every warp reading all partials, which hammers the same L2 lines 12x harder)
__device__ __forceinline__ void grid_sum2(const double* part, int nparts, double& a, double& b, double* red) {
  a = 0.0;
  b = 0.0;
  for (int i = threadIdx.x; i < nparts && threadIdx.x < NTC; i += NTC) {
    a += __ldcg(part + 2 * i);
    b += __ldcg(part + 2 * i + 1);
  }
  block_sum2(a, b, red);
}

// This CTA's partial pair -> part[2*blockIdx.x .. +1] (warp sums, one block barrier, thread 0
// adds the NW warp sums in warp order and stores)
__device__ __forceinline__ void cta_partial2(double a, double b, double* red, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0 && warp < NW) { red[warp] = a; red[NW + warp] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) { x += red[w]; y += red[NW + w]; }
    part[2 * blockIdx.x] = x;
    part[2 * blockIdx.x + 1] = y;
  }
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

// Dispatch on the per-warp fragment count and A-row dedupe.  Every variant is its own
// non-inlined function: one function holding all variants made ptxas spill the software-
// pipelined operands in every loop.
#define QTT_FB_DISPATCH(FN, nf, dedupe, ...)                                     \
  do {                                                                           \
    if (dedupe) {                                                                \
      switch (nf) {                                                              \
        case 1: ring = FN<1, true>(__VA_ARGS__); break;                     \
        case 2: ring = FN<2, true>(__VA_ARGS__); break;                     \
        case 3: ring = FN<3, true>(__VA_ARGS__); break;                     \
        case 4: ring = FN<4, true>(__VA_ARGS__); break;                     \
        case 5: ring = FN<5, true>(__VA_ARGS__); break;                     \
        case 6: ring = FN<6, true>(__VA_ARGS__); break;                     \
        case 7: ring = FN<7, true>(__VA_ARGS__); break;                     \
        case 8: ring = FN<8, true>(__VA_ARGS__); break;                     \
        case 10: ring = FN<10, true>(__VA_ARGS__); break;                   \
        case 12: ring = FN<12, true>(__VA_ARGS__); break;                   \
        default: ring = FN<16, true>(__VA_ARGS__); break;                   \
      }                                                                          \
    } else {                                                                     \
      switch (nf) {                                                              \
        case 1: ring = FN<1, false>(__VA_ARGS__); break;                    \
        case 2: ring = FN<2, false>(__VA_ARGS__); break;                    \
        case 3: ring = FN<3, false>(__VA_ARGS__); break;                    \
        case 4: ring = FN<4, false>(__VA_ARGS__); break;                    \
        case 5: ring = FN<5, false>(__VA_ARGS__); break;                    \
        case 6: ring = FN<6, false>(__VA_ARGS__); break;                    \
        case 7: ring = FN<7, false>(__VA_ARGS__); break;                    \
        case 8: ring = FN<8, false>(__VA_ARGS__); break;                    \
        case 10: ring = FN<10, false>(__VA_ARGS__); break;                  \
        case 12: ring = FN<12, false>(__VA_ARGS__); break;                  \
        default: ring = FN<16, false>(__VA_ARGS__); break;                  \
      }                                                                          \
    }                                                                            \
  } while (0)

// ---- phase 1: t2 <- Bop . v^T.  CTA c owns fragment rows [c*FR/G, (c+1)*FR/G) in
// row blocks of <= p1_rb fragments, times column blocks of <= p1_cb fragments.
template <int NF, bool DEDUPE>
__device__ __noinline__ tmafb::Ring phase1_t(const CGTmaArgs& a, const CUtensorMap* mv, tmafb::Ring ring) {
  const int M = a.lb * a.m * a.R1, N = a.rk, K = a.lk * a.n;
  const int FR = (M + 7) / 8, FC = (N + 7) / 8;
  const int KT = (K + 15) / 16;
  const int G = gridDim.x, c = blockIdx.x;
  const int r0 = (int)((long long)c * FR / G), r1 = (int)((long long)(c + 1) * FR / G);
  const int RB = a.p1_rb, CB = a.p1_cb;
  const int nrb = (r1 - r0 + RB - 1) / RB, ncb = (FC + CB - 1) / CB;
  const tmafb::Boxes bx{&a.map_bop, mv, a.box1_a, a.box1_b};
  // p1_frun > 0: every CTA owns its exact 1/G share of ALL fragments (a row-major run), streamed
  // as p1_frun regions (one while the share fits the warps' accumulators)
  const long long Fall = (long long)FR * FC;
  const int fb_all = (int)(Fall * c / G), fe_all = (int)(Fall * (c + 1) / G);
  auto get = [&](int i) {
    tmafb::Region g;
    g.kb = 0;
    g.ke = KT;
    if (a.p1_frun) {  // chunk i of this CTA's fragment run (p1_frun chunks of equal length)
      const int chunk = (fe_all - fb_all + a.p1_frun - 1) / a.p1_frun;
      const int fb = fb_all + i * chunk, fe = min(fe_all, fb + chunk);
      const int fr0 = fb / FC, fr1 = (fe - 1) / FC + 1;
      g.m0 = fr0 * 8;
      g.mrows = (fr1 - fr0) * 8;
      g.n0 = 0;
      g.ncols = FC * 8;
      g.fb = fb - fr0 * FC;
      g.fe = fe - fr0 * FC;
      return g;
    }
    const int rb = i / ncb, cb = i - (i / ncb) * ncb;
    g.m0 = (r0 + rb * RB) * 8;
    g.mrows = min(RB, r1 - r0 - rb * RB) * 8;
    g.n0 = cb * CB * 8;
    g.ncols = min(CB, FC - cb * CB) * 8;
    g.fb = 0;
    g.fe = 0;
    return g;
  };
  const int R1 = a.R1, rk = a.rk;
  const long long K3p = a.K3p;
  double* t2 = a.t2;
  auto epi = [&](const tmafb::Region& g, const auto& fr, const auto& acc) {
    tmafb::store(g, fr, acc, M, N, [&](int r) {
      const int xm = r / R1, bb = r - xm * R1;
      return t2 + xm * K3p + (long long)bb * rk;
    });
  };
  int nreg = r1 > r0 ? nrb * ncb : 0;
  if (a.p1_frun) {  // non-empty chunks
    const int len = fe_all - fb_all, chunk = (len + a.p1_frun - 1) / a.p1_frun;
    nreg = len > 0 ? (len + chunk - 1) / chunk : 0;
  }
  tmafb::stream<NF, DEDUPE>(ring, bx, nreg, get, epi);
  return ring;
}

__device__ __forceinline__ void phase1(const CGTmaArgs& a, const CUtensorMap* mv, tmafb::Ring& ring) {
  QTT_FB_DISPATCH(phase1_t, a.p1_nf, a.p1_dedupe != 0, a, mv, ring);
}

// ---- phase 2 (split-K): part3[s][Y][(X,m)] = phir[Y, slice s] . t2[(X,m), slice s];
// one region per CTA: fragment-block tile x K slice.
template <int NF, bool DEDUPE>
__device__ __noinline__ tmafb::Ring phase2_t(const CGTmaArgs& a, tmafb::Ring ring) {
  const int M = a.rb, N = a.lb * a.m, K = a.R1 * a.rk;
  const int FR = (M + 7) / 8, FC = (N + 7) / 8;
  const int KT = (K + 15) / 16;
  const int S = a.S3, ktp = a.kt_per3;
  const int RB = a.p2_rb, CB = a.p2_cb;
  const int ntc = (FC + CB - 1) / CB, ntr = (FR + RB - 1) / RB;
  const int items = ntr * ntc * S;
  const tmafb::Boxes bx{&a.map_phir, &a.map_t2, a.box2_a, a.box2_b};
  const int it0 = blockIdx.x;
  auto get = [&](int i) {
    const int it = it0 + i * gridDim.x;
    const int s = it % S, tile = it / S;
    const int tr = tile / ntc, tc = tile - (tile / ntc) * ntc;
    tmafb::Region g;
    g.m0 = tr * RB * 8;
    g.mrows = min(RB, FR - tr * RB) * 8;
    g.n0 = tc * CB * 8;
    g.ncols = min(CB, FC - tc * CB) * 8;
    g.kb = s * ktp;
    g.ke = min(KT, g.kb + ktp);
    g.fb = 0;
    g.fe = 0;
    return g;
  };
  const long long dim = a.dim;
  double* part3 = a.part3;
  auto epi = [&](const tmafb::Region& g, const auto& fr, const auto& acc) {
    double* P = part3 + (long long)(g.kb / ktp) * dim;
    tmafb::store(g, fr, acc, M, N, [&](int r) { return P + (long long)r * N; });
  };
  const int mine = items > it0 ? (items - 1 - it0) / (int)gridDim.x + 1 : 0;
  tmafb::stream<NF, DEDUPE>(ring, bx, mine, get, epi);
  return ring;
}

__device__ __forceinline__ void phase2(const CGTmaArgs& a, tmafb::Ring& ring) {
  QTT_FB_DISPATCH(phase2_t, a.p2_nf, a.p2_dedupe != 0, a, ring);
}

__device__ void matvec(const CGTmaArgs& a, const CUtensorMap* mv, tmafb::Ring& ring, cg::grid_group& grid,
                       unsigned long long& tp) {
  const unsigned long long ts = a.cta_ns != nullptr ? gtimer() : 0;
  ring.dbg_slot = 0;
  phase1(a, mv, ring);
  if (a.cta_ns != nullptr && threadIdx.x == 0) a.cta_ns[blockIdx.x] += gtimer() - ts;
  fence_proxy_global();
  grid.sync();
  phase_mark(a, 1, tp);
  const unsigned long long ts2 = a.cta_ns != nullptr ? gtimer() : 0;
  ring.dbg_slot = 1;
  phase2(a, ring);
  if (a.cta_ns != nullptr && threadIdx.x == 0) a.cta_ns[gridDim.x + blockIdx.x] += gtimer() - ts2;
  grid.sync();
  phase_mark(a, 2, tp);
}

// Split-K reduction of this CTA's slice [e0, e1), NT elements at a time: warp w
// sums partials k = w, w+NW, ... for every element of the chunk with all loads in
// flight together, then the NW warp sums are added in warp order through shared
// memory (deterministic).  f(e, q) runs on the thread owning element e.
template <class F>
__device__ __forceinline__ void reduce_slice(const CGTmaArgs& a, long long e0, long long e1, double* sred, F&& f) {
  constexpr int W = NW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S3;
  const long long dim = a.dim;
  const double* part = a.part3;
  for (long long c0 = e0; c0 < e1; c0 += NTC) {
    const int cnt = (int)min((long long)NTC, e1 - c0);
    if (warp < W) {
      double acc[W];
#pragma unroll
      for (int ch = 0; ch < W; ++ch) acc[ch] = 0.0;
      // two partials per pass with all their loads issued before the adds (same add order)
      for (int k = warp; k < S; k += 2 * W) {
        const double* pk = part + k * dim + c0;
        const bool two = k + W < S;
        double v0[W], v1[W];
#pragma unroll
        for (int ch = 0; ch < W; ++ch) {
          const int el = ch * 32 + lane;
          v0[ch] = el < cnt ? __ldcg(pk + el) : 0.0;
          v1[ch] = (two && el < cnt) ? __ldcg(pk + W * dim + el) : 0.0;
        }
#pragma unroll
        for (int ch = 0; ch < W; ++ch) {
          if (ch * 32 + lane < cnt) {
            acc[ch] += v0[ch];
            if (two) acc[ch] += v1[ch];
          }
        }
      }
#pragma unroll
      for (int ch = 0; ch < W; ++ch) sred[warp * NTC + ch * 32 + lane] = acc[ch];
    }
    __syncthreads();
    if ((int)threadIdx.x < cnt) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < W; ++w) s += sred[w * NTC + threadIdx.x];
      f(c0 + threadIdx.x, s);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(NT, 1) cg_tma_kernel(const __grid_constant__ CGTmaArgs a) {
  extern __shared__ unsigned char smem_raw[];
  __shared__ double red[2 * NW + 4];
  cg::grid_group grid = cg::this_grid();
  const long long n = a.dim;
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long e0 = blockIdx.x * per, e1 = min(n, e0 + per);
  unsigned long long mv_ns = 0, t0 = 0, tp = gtimer();
  const bool timer = (blockIdx.x == 0 && threadIdx.x == 0);
  tmafb::Ring ring = tmafb::ring_init(smem_raw, a.stage_stride, a.stages);
  if (a.cta_ns != nullptr) ring.dbg = a.cta_ns + 3 * gridDim.x;  // timeline of CTA 0's streams
  if (threadIdx.x == 0) {
    tma::prefetch_map(&a.map_bop);
    tma::prefetch_map(&a.map_z);
    tma::prefetch_map(&a.map_phir);
    tma::prefetch_map(&a.map_t2);
  }
  if (a.cta_ns != nullptr && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.cta_ns[2 * gridDim.x + blockIdx.x] = smid;
  }
  grid.sync();

  // ---- r = b - A x0 (only when x0 has a nonzero entry, as scipy's `x.any()`)
  if (a.xany) {
    if (timer) t0 = gtimer();
    matvec(a, &a.map_x, ring, grid, tp);
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
  double* sred = reinterpret_cast<double*>(ring.base);  // ring is idle between GEMM phases
  if (a.xany)
    reduce_slice(a, e0, e1, sred, init_r);
  else
    for (long long e = e0 + threadIdx.x; e < e1 && threadIdx.x < NTC; e += NTC) init_r(e, 0.0);
  fence_proxy_global();
  cta_partial2(rr, rz, red, a.red);
  grid.sync();
  grid_sum2(a.red, gridDim.x, rr, rz, red);
  double rho = rz, rnorm = sqrt(rr);
  int it = 0;
  double* red_pq = a.red + 2 * gridDim.x;

  // SciPy's recurrence with the search direction folded into the matvec: w = A z,
  // then q = w + beta q (= A p since p = z + beta p) and p = z + beta p in the
  // reduction phase -- one grid barrier per iteration less than q = A p after a
  // separate p update.  (Identical in exact arithmetic; p = z, q = A z when beta = 0.)
  double beta = 0.0;
  while (!(rnorm < a.atol) && it < a.maxiter) {
    if (timer) t0 = gtimer();
    matvec(a, &a.map_z, ring, grid, tp);
    double pq = 0.0, dummy = 0.0;
    const double bq = beta;
    // this thread's element of a one-chunk slice: its q, z, p loads overlap the partial sums
    // (first iteration: beta = 0 and q/p are never read -- q is uninitialised pool memory,
    // where 0 * NaN would poison the solve; wi + 0 * q == wi for every finite q anyway)
    const long long me = e0 + threadIdx.x;
    const bool pre = (e1 - e0) <= NTC && me < e1 && threadIdx.x < NTC;
    const bool first = bq == 0.0;
    double q0 = 0.0, z0 = 0.0, p0 = 0.0;
    if (pre) {
      z0 = a.z[me];
      if (!first) {
        q0 = a.q[me];
        p0 = a.p[me];
      }
    }
    reduce_slice(a, e0, e1, sred, [&](long long e, double wi) {
      const bool hit = pre && e == me;
      const double qi = first ? wi : wi + bq * (hit ? q0 : a.q[e]);
      const double zi = hit ? z0 : a.z[e];
      const double pi = first ? zi : zi + bq * (hit ? p0 : a.p[e]);
      a.q[e] = qi;
      a.p[e] = pi;
      pq += pi * qi;
    });
    cta_partial2(pq, dummy, red, red_pq);
    grid.sync();
    phase_mark(a, 3, tp);
    if (timer) mv_ns += gtimer() - t0;
    grid_sum2(red_pq, gridDim.x, pq, dummy, red);
    const double alpha = rho / pq;
    rr = 0.0;
    rz = 0.0;
    for (long long e = e0 + threadIdx.x; e < e1 && threadIdx.x < NTC; e += NTC) {
      a.x[e] += alpha * a.p[e];
      const double ri = a.r[e] - alpha * a.q[e];
      a.r[e] = ri;
      const double zi = ri * a.invd[e];
      a.z[e] = zi;
      rr += ri * ri;
      rz += ri * zi;
    }
    fence_proxy_global();  // z feeds the next matvec through TMA
    cta_partial2(rr, rz, red, a.red);
    grid.sync();
    phase_mark(a, 4, tp);
    grid_sum2(a.red, gridDim.x, rr, rz, red);
    ++it;
    rnorm = sqrt(rr);
    if (rnorm < a.atol || it >= a.maxiter) break;
    beta = rz / rho;
    rho = rz;
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

// the ring also serves as scratch for the split-K reduction (NW x NTC doubles)
constexpr size_t SMEM_MAX = 224 * 1024;  // + static shared memory <= the 227 KB opt-in limit
size_t cg_tma_smem(int stride, int nst) {
  return std::max((size_t)nst * stride, (size_t)NW * NTC * sizeof(double)) + tmafb::HEADER + 1024 + 4096;
}
// Ring depth: 4 stages (look-ahead 2 k-tiles) when they fit, at least 3 (QTT_TMA_STAGES
// overrides).  Measured at r = 100, R = 31 / 52 (both GEMM phases of one matvec, us): 3 stages
// 18.96 / 29.46, 4 stages 18.63 / 29.05, 6 stages 18.98 / 29.46, 8 stages 19.23 / 29.81 -- a
// deeper prologue burst only delays the first k-tile (phase 2 first data 1.5 -> 2.9 us).
int cg_tma_stages(int stride) {
  int want = 4;
  if (const char* e = std::getenv("QTT_TMA_STAGES")) want = std::atoi(e);
  const int fit = (int)((SMEM_MAX - tmafb::HEADER - 1024 - 4096) / (size_t)stride);
  return std::max(3, std::min({want, fit, tmafb::MAX_STAGES}));
}

int cg_tma_grid(int device) {
  static PerDevice<int> cache(-1);
  int& cached = cache.at(device);
  if (cached > 0) return cached;
  const size_t smem = std::getenv("QTT_TMA_ATTR_KB") ? (size_t)std::atoi(std::getenv("QTT_TMA_ATTR_KB")) * 1024
                                                     : SMEM_MAX;
  QTT_CUDA(cudaFuncSetAttribute(cg_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0, sms = 0;
  QTT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_tma_kernel, NT, smem));
  QTT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (per_sm < 1) throw Error(QTT_ERR_CUDA, "cg_tma_kernel cannot be resident (registers/shared memory)");
  cached = sms;
  return cached;
}

CGTmaPlan cg_tma_plan(int lb, int m, int R1, int lk, int n, int rb, int rk, int grid) {
  CGTmaPlan p{};
  constexpr int FMAX = tmafb::MAXF * tmafb::NWARP;  // fragments per region
  // phase 1: M1 x N1, each CTA ~FR/G fragment rows
  const long long M1 = (long long)lb * m * R1;
  const int FR1 = (int)cdiv(M1, 8), FC1 = cdiv(rk, 8);
  p.p1_rb = std::max(1, std::min(32, cdiv(FR1, grid)));
  p.p1_cb = std::max(1, std::min({FC1, FMAX / p.p1_rb, 32, 52 - p.p1_rb}));
  if (const char* e = std::getenv("QTT_TMA_P1")) std::sscanf(e, "%d,%d", &p.p1_rb, &p.p1_cb);
  p.box1_a = p.p1_rb * 8;
  p.box1_b = p.p1_cb * 8;
  p.p1_nf = tmafb::nf_for(p.p1_rb * p.p1_cb);
  // dedupe needs every column block (the last may be narrower) to hold a run in 2 rows
  const int cb1_min = FC1 % p.p1_cb == 0 ? p.p1_cb : FC1 % p.p1_cb;
  p.p1_dedupe = tmafb::dedupe_ok(p.p1_nf, cb1_min) ? 1 : 0;
  // fragment-run dealing: when one region per CTA can hold its 1/G share of all fragments
  // (all columns in one box), CTAs get equal fragment counts instead of whole fragment rows
  p.p1_frun = 0;
  {
    const long long Fall = (long long)FR1 * FC1;
    int fmax = 0, rmax = 1;
    for (int c = 0; c < grid; ++c) {
      const int fb = (int)(Fall * c / grid), fe = (int)(Fall * (c + 1) / grid);
      if (fe <= fb) continue;
      fmax = std::max(fmax, fe - fb);
      rmax = std::max(rmax, (fe - 1) / FC1 - fb / FC1 + 1);
    }
    static const int frun_env = std::getenv("QTT_TMA_FRUN") ? std::atoi(std::getenv("QTT_TMA_FRUN")) : 1;
    // shares beyond 10 fragments per warp (the largest variant that neither spills nor leaves a
    // tail region half empty: C5, rank 196, 430 fragments per CTA) are cut into equal chunks
    const int chunks = fmax > 0 ? cdiv(fmax, 10 * tmafb::NWARP) : 1;
    const int cmax = fmax > 0 ? cdiv(fmax, chunks) : 0;
    int rmax_c = 1;
    for (int c = 0; c < grid && chunks > 1; ++c) {
      const int fb = (int)(Fall * c / grid), fe = (int)(Fall * (c + 1) / grid);
      const int chunk = cdiv(fe - fb, chunks);
      for (int i = 0; i < chunks && chunk > 0; ++i) {
        const int b = fb + i * chunk, e = std::min(fe, b + chunk);
        if (e > b) rmax_c = std::max(rmax_c, (e - 1) / FC1 - b / FC1 + 1);
      }
    }
    if (chunks == 1) rmax_c = rmax;
    if (frun_env && FC1 <= 32 && fmax > 0 && chunks <= 16 && rmax_c <= 32 && (rmax_c + FC1) * 8 * 128 <= 48 * 1024) {
      p.p1_frun = chunks;
      p.p1_cb = FC1;
      p.box1_a = rmax_c * 8;
      p.box1_b = FC1 * 8;
      p.p1_nf = tmafb::nf_for(cmax);
      p.p1_dedupe = tmafb::dedupe_ok(p.p1_nf, FC1) ? 1 : 0;
    }
  }
  // phase 2: split-K; choose the fragment-block tiling and split count that
  // minimise per-CTA DMMAs plus the split-K partial traffic
  const int FR3 = cdiv(rb, 8), FC3 = cdiv(lb * m, 8);
  const int KT3 = cdiv(R1 * rk, 16);
  double best = 1e300;
  for (int tr = cdiv(FR3, 32); tr <= FR3; ++tr) {
    const int RB = cdiv(FR3, tr);
    for (int tc = 1; tc <= FC3; ++tc) {
      const int CB = cdiv(FC3, tc);
      if (RB * CB > FMAX || RB > 32 || CB > 32 || RB + CB > 52) continue;
      const int T = cdiv(FR3, RB) * cdiv(FC3, CB);
      if (T > grid) continue;
      const int want = std::max(1, std::min(grid / T, std::max(1, KT3 / 2)));
      const int ktp = cdiv(KT3, want);
      const int S = cdiv(KT3, ktp);
      // per-CTA time in DMMA-clock units: NF-quantized fragments x k-tiles x (4 k-steps x
      // 3 warps x 16 clk), + ~2.5 us first-data latency, + the partial store/reload
      // per k-tile: DMMA issue (NF x 4 k-steps x 3 warps x 16 clk) or the L2->SMEM
      // operand stream ((RB + CB) x 8 rows x 128 B at ~24 B/clk per SM), whichever is longer
      // (or the ~2 us TMA round trip spread over the ring depth)
      // (the latency term keeps the 4-stage ring's value: the split it selects fixes the
      // summation order of q, and with it the solve's trajectory)
      const int nst = 4;
      // (the model keeps the even fragment counts it was tuned with: its choice of split fixes
      // the summation order of q)
      const int per12 = cdiv(RB * CB, tmafb::NWARP);
      const int nf_model = per12 <= 4 ? 4 : per12 <= 6 ? 6 : per12 <= 8 ? 8 : per12 <= 10 ? 10 : per12 <= 12 ? 12 : 16;
      const double per_kt = std::max({(double)nf_model * 4.0 * 48.0, (RB + CB) * 8.0 * 128.0 / 24.0,
                                      4000.0 / (nst - 1)});
      const double dmma = per_kt * ktp;
      const double traffic = (double)S * rb * lb * m * 8.0 * 2.0 / 4.0e12 * 1.965e9;  // write+read at ~4 TB/s
      const double c = dmma + 5000.0 + traffic;
      if (c < best * 0.999) {
        best = c;
        p.p2_rb = RB;
        p.p2_cb = CB;
        p.S3 = S;
        p.kt_per3 = ktp;
      }
    }
  }
  if (const char* e = std::getenv("QTT_TMA_P2")) {  // "rb,cb,S": force the phase-2 tiling (tuning)
    int S = 0;
    if (std::sscanf(e, "%d,%d,%d", &p.p2_rb, &p.p2_cb, &S) == 3 && S > 0) {
      p.kt_per3 = cdiv(KT3, S);
      p.S3 = cdiv(KT3, p.kt_per3);
    }
  }
  p.box2_a = p.p2_rb * 8;
  p.box2_b = p.p2_cb * 8;
  p.p2_nf = tmafb::nf_for(p.p2_rb * p.p2_cb);
  const int cb2_min = FC3 % p.p2_cb == 0 ? p.p2_cb : FC3 % p.p2_cb;
  p.p2_dedupe = tmafb::dedupe_ok(p.p2_nf, cb2_min) ? 1 : 0;
  const int bytes = std::max(p.box1_a + p.box1_b, p.box2_a + p.box2_b) * 128;
  p.stage_stride = cdiv(bytes, 1024) * 1024;
  p.stages = cg_tma_stages(p.stage_stride);
  (void)lk;
  (void)n;
  return p;
}

void cg_tma_launch(const CGTmaArgs& a, int grid, cudaStream_t s) {
  void* args[] = {(void*)&a};
  QTT_CUDA(cudaLaunchCooperativeKernel((void*)cg_tma_kernel, dim3(grid), dim3(NT), args,
                                       cg_tma_smem(a.stage_stride, a.stages), s));
  QTT_CHECK_LAUNCH();
}

void transpose_2d(const double* in, double* out, long long rows, long long cols, cudaStream_t s) {
  dim3 g((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32));
  transpose_kernel<<<g, dim3(32, 8), 0, s>>>(in, out, rows, cols);
  QTT_CHECK_LAUNCH();
}

}  // namespace qtt
