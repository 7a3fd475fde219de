// Blocked Householder QR for large unfoldings (dgeqrf-style, right-looking):
// a cooperative panel kernel factors nb = 64 columns (LAPACK dlarfg signs), a small
// kernel forms the block reflector T (dlarft), and the trailing matrix is updated
// with three DMMA GEMMs  C -= V (T^T (V^T C)).  Used where the single-CTA kernel of
// linalg.cu would serialize: the rank R*r + r_f unfoldings of the residual
// certification sweep (amen.py:87-99 via tt.py:362-371) and large roundings.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "contract.cuh"
#include "gemm.cuh"
#include "linalg.cuh"
#include "qr_blocked.cuh"

namespace cg = cooperative_groups;

namespace qtt {
namespace {

constexpr int PNT = 256;  // threads per panel CTA
constexpr int NB = 64;    // panel width

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < PNT / 32 ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  const double out = red[32];
  __syncthreads();
  return out;
}

struct PanelArgs {
  double* W;  // column-major, leading dimension ld
  long long ld;
  int m;      // total rows
  int j0;     // first panel column (= first panel row)
  int jb;     // panel width
  double* tau;
  double* red;  // gridDim * (NB + 1) doubles
  unsigned long long* tl;  // optional (QTT_DEBUG=2): CTA 0 per-step ns accumulators [5]
  // cluster panel only (optional): write the unit lower trapezoid V (mrows x jb, column-
  // major) and the block reflector T (jb x jb row-major upper; dlarft forward columnwise),
  // also into T_big at (tb_off, tb_off) with leading dimension ldtb when Tb != nullptr
  double* Vb = nullptr;
  double* T = nullptr;
  double* Tb = nullptr;
  long long ldtb = 0;
  int tb_off = 0;
};

__device__ __forceinline__ unsigned long long qr_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Factor W[j0:m, j0:j0+jb].  Rows j0..m-1 are split over the CTAs; per column two
// grid barriers: one after the partial norms, one after the partial dot products.
__global__ void __launch_bounds__(PNT) panel_kernel(PanelArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[40];
  __shared__ double sw[NB];
  __shared__ double sbeta[NB];
  const int G = gridDim.x;
  const int rows = a.m - a.j0;
  const int chunk = (rows + G - 1) / G;
  const int r0 = a.j0 + blockIdx.x * chunk, r1 = min(a.m, r0 + chunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* W = a.W;
  const long long ld = a.ld;
  for (int j = 0; j < a.jb; ++j) {
    const int col = a.j0 + j, rj = a.j0 + j;
    double* v = W + col * ld;
    double part = 0.0;
    for (int i = max(r0, rj + 1) + threadIdx.x; i < r1; i += PNT) part += v[i] * v[i];
    part = block_sum(part, red);
    if (threadIdx.x == 0) a.red[blockIdx.x * (NB + 1)] = part;
    grid.sync();
    double xn = 0.0;
    for (int b = threadIdx.x; b < G; b += PNT) xn += __ldcg(a.red + b * (NB + 1));
    const double xnorm2 = block_sum(xn, red);
    const double alpha = __ldcg(v + rj);
    double t = 0.0, beta = alpha, scal = 1.0;
    if (xnorm2 > 0.0) {  // dlarfg
      beta = -copysign(hypot(alpha, sqrt(xnorm2)), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
      for (int i = max(r0, rj + 1) + threadIdx.x; i < r1; i += PNT) v[i] *= scal;
    }
    if (threadIdx.x == 0) sbeta[j] = beta;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.tau[col] = t;
    __syncthreads();
    const bool own_rj = (rj >= r0 && rj < r1);
    // partial w_c = v^T W[:, c] for the remaining panel columns
    const int nrem = a.jb - j - 1;
    if (t != 0.0 && nrem > 0) {
      for (int cc = warp; cc < nrem; cc += PNT / 32) {
        const double* wc = W + (long long)(col + 1 + cc) * ld;
        double s = 0.0;
        for (int i = max(r0, rj + 1) + lane; i < r1; i += 32) s += v[i] * wc[i];
        s = warp_sum(s);
        if (lane == 0) a.red[blockIdx.x * (NB + 1) + 1 + cc] = s + (own_rj ? wc[rj] : 0.0);
      }
    }
    grid.sync();
    if (t != 0.0 && nrem > 0) {
      for (int cc = warp; cc < nrem; cc += PNT / 32) {
        double s = 0.0;
        for (int b = lane; b < G; b += 32) s += __ldcg(a.red + b * (NB + 1) + 1 + cc);
        s = warp_sum(s);
        if (lane == 0) sw[cc] = s * t;
      }
      __syncthreads();
      for (int cc = 0; cc < nrem; ++cc) {
        double* wc = W + (long long)(col + 1 + cc) * ld;
        const double w = sw[cc];
        for (int i = max(r0, rj + 1) + threadIdx.x; i < r1; i += PNT) wc[i] -= w * v[i];
        if (own_rj && threadIdx.x == 0) wc[rj] -= w;
      }
      __syncthreads();
    }
  }
  // write the R diagonal (betas) now that no column needs its alpha any more
  __syncthreads();
  for (int j = threadIdx.x; j < a.jb; j += PNT) {
    const int rj = a.j0 + j;
    if (rj >= r0 && rj < r1) W[(long long)(a.j0 + j) * ld + rj] = sbeta[j];
  }
}

// Vb (mrows x jb, column-major) = unit lower trapezoid of the panel; T (jb x jb,
// row-major, upper) from tau and Gram = Vb^T Vb (dlarft, forward columnwise).
__global__ void build_v_kernel(const double* W, long long ld, int j0, int mrows, int jb, double* Vb) {
  const long long total = (long long)mrows * jb;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e / mrows), i = (int)(e % mrows);
    Vb[e] = i > j ? W[(long long)(j0 + j) * ld + j0 + i] : (i == j ? 1.0 : 0.0);
  }
}

__global__ void build_t_kernel(const double* Gram, const double* tau, int jb, double* T) {
  // T[j][j] = tau_j;  T[0:j, j] = -tau_j T[0:j, 0:j] Gram[0:j, j]
  __shared__ double s[NB][NB + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) s[e / jb][e % jb] = 0.0;
  __syncthreads();
  for (int j = 0; j < jb; ++j) {
    if (threadIdx.x < j) {
      double acc = 0.0;
      for (int p = threadIdx.x; p < j; ++p) acc += s[threadIdx.x][p] * Gram[p * jb + j];
      s[threadIdx.x][j] = -tau[j] * acc;
    }
    if (threadIdx.x == 0) s[j][j] = tau[j];
    __syncthreads();
  }
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) T[e] = s[e / jb][e % jb];
}

constexpr int SMEM_PANEL_DOUBLES = 26 * 1024;

// Same factorization as panel_kernel, with each CTA's row block of the panel staged
// in shared memory and few CTAs (<= 32): the per
// column work is a few smem passes, so the two grid barriers per column dominate
// (cg grid.sync measured 1.2 us vs 2.1-2.5 us for a hand-rolled generation barrier,
// tools/barrier_bench.cu).
__global__ void __launch_bounds__(PNT) panel_smem_kernel(PanelArgs a) {
  extern __shared__ double P[];  // [jb][nloc] column-major
  __shared__ double red[40];
  __shared__ double sw[NB];
  __shared__ double sbeta[NB];
  const int G = gridDim.x;
  const int rows = a.m - a.j0;
  const int chunk = (rows + G - 1) / G;
  const int r0 = a.j0 + blockIdx.x * chunk, r1 = min(a.m, r0 + chunk);
  const int nloc = max(0, r1 - r0);
  const int ldp = nloc | 1;  // odd column pitch: no bank conflicts across columns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* W = a.W;
  const long long ld = a.ld;
  for (int e = threadIdx.x; e < nloc * a.jb; e += PNT) {
    const int c = e / nloc, i = e % nloc;
    P[c * ldp + i] = W[(long long)(a.j0 + c) * ld + r0 + i];
  }
  __syncthreads();
  // thread layout for the per-column partial dot products / reductions: column cc
  // (< NB) times KS = PNT/NB sub-ranges, combined through shared memory in fixed order
  constexpr int KS = PNT / NB;
  __shared__ double sred[KS][NB];
  const int tcc = threadIdx.x % NB, tsub = threadIdx.x / NB;
  const bool tl = a.tl != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long tc = tl ? qr_clock() : 0;
  auto mark = [&](int i) {
    if (tl) {
      const unsigned long long now = qr_clock();
      a.tl[i] += now - tc;
      tc = now;
    }
  };
  for (int j = 0; j < a.jb; ++j) {
    const int rj = a.j0 + j;
    double* v = P + j * ldp;  // local rows r0..r1
    const int ib = max(0, rj + 1 - r0);  // first local row strictly below rj
    double part = 0.0;
    for (int i = ib + threadIdx.x; i < nloc; i += PNT) part += v[i] * v[i];
    part = block_sum(part, red);
    const bool own_rj = (rj >= r0 && rj < r1);
    if (threadIdx.x == 0) {
      a.red[blockIdx.x * (NB + 2)] = part;
      a.red[blockIdx.x * (NB + 2) + NB + 1] = own_rj ? v[rj - r0] : 0.0;  // alpha
    }
    mark(0);
    cg::this_grid().sync();
    mark(1);
    double xn = 0.0, al = 0.0;
    for (int b = threadIdx.x; b < G; b += PNT) {
      xn += __ldcg(a.red + b * (NB + 2));
      al += __ldcg(a.red + b * (NB + 2) + NB + 1);
    }
    // one two-value block reduction (exactly one CTA contributed alpha)
    xn = warp_sum(xn);
    al = warp_sum(al);
    if (lane == 0) { red[warp] = xn; red[16 + warp] = al; }
    __syncthreads();
    double xnorm2 = 0.0, alpha = 0.0;
#pragma unroll
    for (int w = 0; w < PNT / 32; ++w) { xnorm2 += red[w]; alpha += red[16 + w]; }
    double t = 0.0, beta = alpha, scal = 1.0;
    if (xnorm2 > 0.0) {  // dlarfg
      beta = -copysign(hypot(alpha, sqrt(xnorm2)), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
      for (int i = ib + threadIdx.x; i < nloc; i += PNT) v[i] *= scal;
    }
    if (threadIdx.x == 0) sbeta[j] = beta;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.tau[rj] = t;
    __syncthreads();
    const int nrem = a.jb - j - 1;
    if (t != 0.0 && nrem > 0) {  // local partial dots  v . w_c  (+ w_c[rj] for the unit head)
      double s = 0.0;
      if (tcc < nrem) {
        const double* wc = P + (j + 1 + tcc) * ldp;
        const int len = (nloc - ib + KS - 1) / KS;
        const int i0 = ib + tsub * len, i1 = min(nloc, i0 + len);
        for (int i = i0; i < i1; ++i) s += v[i] * wc[i];
      }
      sred[tsub][tcc] = s;
      __syncthreads();
      if (threadIdx.x < nrem) {
        double d = 0.0;
#pragma unroll
        for (int k = 0; k < KS; ++k) d += sred[k][threadIdx.x];
        const double* wc = P + (j + 1 + threadIdx.x) * ldp;
        a.red[blockIdx.x * (NB + 2) + 1 + threadIdx.x] = d + (own_rj ? wc[rj - r0] : 0.0);
      }
    }
    mark(2);
    cg::this_grid().sync();
    mark(3);
    if (t != 0.0 && nrem > 0) {
      {  // sum the G partials of each column: KS interleaved sub-ranges per column, all
         // loads independent (one L2 round trip), combined in fixed order
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (tcc < nrem) {
          const double* base = a.red + 1 + tcc;
          int b = tsub;
          for (; b + 3 * KS < G; b += 4 * KS) {
            s0 += __ldcg(base + (long long)b * (NB + 2));
            s1 += __ldcg(base + (long long)(b + KS) * (NB + 2));
            s2 += __ldcg(base + (long long)(b + 2 * KS) * (NB + 2));
            s3 += __ldcg(base + (long long)(b + 3 * KS) * (NB + 2));
          }
          for (; b < G; b += KS) s0 += __ldcg(base + (long long)b * (NB + 2));
        }
        __syncthreads();  // sred reuse
        sred[tsub][tcc] = (s0 + s1) + (s2 + s3);
        __syncthreads();
        if (threadIdx.x < nrem) {
          double d = 0.0;
#pragma unroll
          for (int k = 0; k < KS; ++k) d += sred[k][threadIdx.x];
          sw[threadIdx.x] = d * t;
        }
      }
      __syncthreads();
      if (tcc < nrem) {  // same (column, row-range) layout as the dots: no index division
        double* wc = P + (j + 1 + tcc) * ldp;
        const double w = sw[tcc];
        const int len = (nloc - ib + KS - 1) / KS;
        const int i0 = ib + tsub * len, i1 = min(nloc, i0 + len);
        for (int i = i0; i < i1; ++i) wc[i] -= w * v[i];
        if (tsub == 0 && own_rj) wc[rj - r0] -= w;
      }
      __syncthreads();
    }
    mark(4);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < a.jb; j += PNT) {
    const int rj = a.j0 + j;
    if (rj >= r0 && rj < r1) P[j * ldp + (rj - r0)] = sbeta[j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nloc * a.jb; e += PNT) {
    const int c = e / nloc, i = e % nloc;
    W[(long long)(a.j0 + c) * ld + r0 + i] = P[c * ldp + i];
  }
}

// ---- V and T of a factored panel (replaces build_v + V^T V + dlarft launches): P holds
// this CTA's rows of the factored panel, column-major with pitch ldp; on exit a.Vb (unit
// lower trapezoid, mrows x jb column-major) and a.T (dlarft forward columnwise) are written.
// Must be called by every CTA of the cluster (it contains cluster barriers).
template <int NTH>
__device__ void panel_emit_vt(const PanelArgs& a, double* P, int ldp, int nloc, int r0, cg::cluster_group& cl) {
  const int G = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  __syncthreads();
  const int mrows = a.m - a.j0, jb = a.jb;
  for (int e = threadIdx.x; e < nloc * jb; e += NTH) {  // P -> V in place, and V out
    const int c = e / nloc, i = e % nloc;
    const int pr = r0 - a.j0 + i;  // row inside the panel
    const double v = pr > c ? P[c * ldp + i] : (pr == c ? 1.0 : 0.0);
    P[c * ldp + i] = v;
    a.Vb[(long long)c * mrows + pr] = v;
  }
  __syncthreads();
  // partial Gram of this CTA's rows: thread owns a 4x4 block of the 64x64 index space;
  // Gp / Gs / Ts live in the (now free) dynamic panel buffer, sized for them at launch
  double (*Gp)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(P);
  double (*Gs)[NB + 1] = Gp + NB;
  double (*Ts)[NB + 1] = Gp + 2 * NB;
  {
    const int tg = threadIdx.x & 255;  // 256-thread Gram layout (extra threads idle)
    const int p0 = 4 * (tg >> 4), q0 = 4 * (tg & 15);
    const bool gact = threadIdx.x < 256;
    double g[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) g[x][y] = 0.0;
    if (gact && p0 < jb && q0 < jb && q0 + 3 >= p0) {  // blocks touching the upper triangle
      for (int i = 0; i < nloc; ++i) {
        double vp[4], vq[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          vp[x] = p0 + x < jb ? P[(p0 + x) * ldp + i] : 0.0;
          vq[x] = q0 + x < jb ? P[(q0 + x) * ldp + i] : 0.0;
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) g[x][y] = fma(vp[x], vq[y], g[x][y]);
      }
    }
    __syncthreads();  // every thread is done reading V from P
    if (gact)
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) Gp[p0 + x][q0 + y] = g[x][y];
  }
  cl.sync();
  if (rank == 0) {  // sum the partials in rank order, then the dlarft recursion in shared memory
    for (int e = threadIdx.x; e < jb * jb; e += NTH) {
      const int p = e / jb, q = e % jb;
      double sum = 0.0;
      if (p < q)
        for (int r = 0; r < G; ++r) sum += cl.map_shared_rank(&Gp[0][0], r)[p * (NB + 1) + q];
      Gs[p][q] = sum;
      Ts[p][q] = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < jb; ++j) {  // T[j][j] = tau_j;  T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]
      const double tj = a.tau[a.j0 + j];
      if ((int)threadIdx.x < j) {
        double acc = 0.0;
        for (int q = threadIdx.x; q < j; ++q) acc = fma(Ts[threadIdx.x][q], Gs[q][j], acc);
        Ts[threadIdx.x][j] = -tj * acc;
      }
      if (threadIdx.x == 0) Ts[j][j] = tj;
      __syncthreads();
    }
    for (int e = threadIdx.x; e < jb * jb; e += NTH) {
      const int p = e / jb, q = e % jb;
      a.T[e] = Ts[p][q];
      if (a.Tb) a.Tb[(long long)(a.tb_off + p) * a.ldtb + a.tb_off + q] = Ts[p][q];
    }
  }
  cl.sync();  // no CTA leaves while rank 0 may still read its shared memory
}


// Panel factorization inside ONE thread-block cluster (up to 16 CTAs on one GPC):
// the per-column reductions go through distributed shared memory and the two
// barriers per column are hardware cluster barriers, instead of L2 round trips and
// grid-wide barriers of 148 CTAs (tools: QTT_DEBUG=2 panel timeline, ~9 us/column).
// Each CTA keeps its row block of the panel (<= ~200 KB) in shared memory.
__global__ void __launch_bounds__(PNT) panel_cluster_kernel(PanelArgs a) {
  extern __shared__ double P[];  // [jb][nloc] column-major
  __shared__ double red[40];
  __shared__ double dots[NB];    // this CTA's partial dots of the current column
  __shared__ double sw[NB];
  __shared__ double sbeta[NB];
  // (column, row-range) thread layout: CW = panel width rounded to 32/64, KS = PNT/CW
  __shared__ double sred[PNT];
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int rows = a.m - a.j0;
  const int chunk = (rows + G - 1) / G;
  const int r0 = a.j0 + rank * chunk, r1 = min(a.m, r0 + chunk);
  const int nloc = max(0, r1 - r0);
  // odd column pitch: lanes of a warp walk consecutive columns at the same row, so an even
  // pitch would put all 32 of them in one shared-memory bank (32-way conflicts)
  const int ldp = nloc | 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int CW = a.jb <= 32 ? 32 : 64, KS = PNT / CW;
  const int tcc = threadIdx.x % CW, tsub = threadIdx.x / CW;
  double* W = a.W;
  const long long ld = a.ld;
  for (int e = threadIdx.x; e < nloc * a.jb; e += PNT) {
    const int c = e / nloc, i = e % nloc;
    P[c * ldp + i] = W[(long long)(a.j0 + c) * ld + r0 + i];
  }
  __syncthreads();
  const bool tl = a.tl != nullptr && rank == 0 && threadIdx.x == 0;
  unsigned long long tc = tl ? qr_clock() : 0;
  auto mark = [&](int i) {
    if (tl) {
      const unsigned long long now = qr_clock();
      a.tl[i] += now - tc;
      tc = now;
    }
  };
  // inboxes: every CTA PUSHES its partials into all CTAs' shared memory before the cluster
  // barrier (remote stores overlap the barrier), so the reductions after it read local smem
  __shared__ double nin[16][2];
  __shared__ double din[16][NB];
  for (int j = 0; j < a.jb; ++j) {
    const int rj = a.j0 + j;
    double* v = P + j * ldp;
    const int ib = max(0, rj + 1 - r0);
    double pn = 0.0;
#pragma unroll 4
    for (int i = ib + threadIdx.x; i < nloc; i += PNT) pn = fma(v[i], v[i], pn);
    pn = block_sum(pn, red);
    const bool own_rj = (rj >= r0 && rj < r1);
    if ((int)threadIdx.x < G) {
      double* dst = cl.map_shared_rank(&nin[0][0], (int)threadIdx.x);
      dst[2 * rank] = pn;
      dst[2 * rank + 1] = own_rj ? v[rj - r0] : 0.0;
    }
    mark(0);
    cl.sync();
    mark(1);
    // every CTA sums the G partials in the same (lane-tree) order: identical result everywhere
    double xnorm2 = 0.0, alpha = 0.0;
    if (warp == 0) {
      double x = 0.0, y = 0.0;
      if (lane < G) {
        x = nin[lane][0];
        y = nin[lane][1];
      }
      x = warp_sum(x);
      y = warp_sum(y);
      if (lane == 0) { red[32] = x; red[33] = y; }
    }
    __syncthreads();
    xnorm2 = red[32];
    alpha = red[33];
    double t = 0.0, beta = alpha, scal = 1.0;
    if (xnorm2 > 0.0) {  // dlarfg
      beta = -copysign(hypot(alpha, sqrt(xnorm2)), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
      for (int i = ib + threadIdx.x; i < nloc; i += PNT) v[i] *= scal;
    }
    if (threadIdx.x == 0) sbeta[j] = beta;
    if (rank == 0 && threadIdx.x == 0) a.tau[rj] = t;
    __syncthreads();
    const int nrem = a.jb - j - 1;
    if (t != 0.0 && nrem > 0) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (tcc < nrem) {
        const double* wc = P + (j + 1 + tcc) * ldp;
        const int len = (nloc - ib + KS - 1) / KS;
        const int i0 = ib + tsub * len, i1 = min(nloc, i0 + len);
        int i = i0;
        for (; i + 3 < i1; i += 4) {
          s0 = fma(v[i], wc[i], s0);
          s1 = fma(v[i + 1], wc[i + 1], s1);
          s2 = fma(v[i + 2], wc[i + 2], s2);
          s3 = fma(v[i + 3], wc[i + 3], s3);
        }
        for (; i < i1; ++i) s0 = fma(v[i], wc[i], s0);
      }
      sred[tsub * CW + tcc] = (s0 + s1) + (s2 + s3);
      __syncthreads();
      if (threadIdx.x < nrem) {
        double d = 0.0;
        for (int k = 0; k < KS; ++k) d += sred[k * CW + threadIdx.x];
        const double* wc = P + (j + 1 + threadIdx.x) * ldp;
        dots[threadIdx.x] = d + (own_rj ? wc[rj - r0] : 0.0);
      }
      __syncthreads();
      for (int e = threadIdx.x; e < G * nrem; e += PNT) {  // push to every CTA's inbox
        const int r = e / nrem, cc = e - r * nrem;
        cl.map_shared_rank(&din[0][0], r)[rank * NB + cc] = dots[cc];
      }
    }
    mark(2);
    cl.sync();
    mark(3);
    if (t != 0.0 && nrem > 0) {
      // sum each column's partials in rank order (same order in every CTA)
      if (threadIdx.x < nrem) {
        double d = 0.0;
        for (int r = 0; r < G; ++r) d += din[r][threadIdx.x];
        sw[threadIdx.x] = d * t;
      }
      __syncthreads();
      if (tcc < nrem) {
        double* wc = P + (j + 1 + tcc) * ldp;
        const double w = sw[tcc];
        const int len = (nloc - ib + KS - 1) / KS;
        const int i0 = ib + tsub * len, i1 = min(nloc, i0 + len);
#pragma unroll 4
        for (int i = i0; i < i1; ++i) wc[i] = fma(-w, v[i], wc[i]);
        if (tsub == 0 && own_rj) wc[rj - r0] -= w;
      }
      __syncthreads();
    }
    mark(4);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < a.jb; j += PNT) {
    const int rj = a.j0 + j;
    if (rj >= r0 && rj < r1) P[j * ldp + (rj - r0)] = sbeta[j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nloc * a.jb; e += PNT) {
    const int c = e / nloc, i = e % nloc;
    W[(long long)(a.j0 + c) * ld + r0 + i] = P[c * ldp + i];
  }
  if (a.T == nullptr) {
    cl.sync();  // no CTA leaves while another may still read its shared memory
    return;
  }
  panel_emit_vt<PNT>(a, P, ldp, nloc, r0, cl);
}

// Register-resident panel (jb <= 32): the same factorization as panel_cluster_kernel, but each
// thread keeps its rows of the panel (RPT rows x 32 columns) in REGISTERS for the whole panel.
// Per column the only shared-memory traffic is the reductions: the partial dot products of the
// reflector with the remaining columns are reduced inside each warp by a transpose-reduction
// (8 columns per pass, 3 halving shuffle steps + 2 butterflies) instead of streaming every
// column of the panel through shared memory twice (the smem kernel is bandwidth-bound there).
constexpr int RJB = 32;
template <int RPT>
__global__ void __launch_bounds__(PNT, 1) panel_reg_kernel(PanelArgs a) {
  extern __shared__ double P[];  // V/T emission scratch (written column by column)
  constexpr int NWW = PNT / 32;
  __shared__ double red2[2 * NWW];
  __shared__ double nin[16][2];
  __shared__ double din[16][RJB];
  __shared__ double wsum[NWW][RJB];
  __shared__ double sw[RJB];
  cg::cluster_group cl = cg::this_cluster();
  const int G = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int rows = a.m - a.j0;
  const int chunk = (rows + G - 1) / G;
  const int r0 = a.j0 + rank * chunk, r1 = min(a.m, r0 + chunk);
  const int nloc = max(0, r1 - r0);
  const int ldp = nloc | 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jb = a.jb;
  double* W = a.W;
  const long long ld = a.ld;
  constexpr int NONE = 0x7fffffff;
  // w[q][0] is always the CURRENT column: the register window shifts left by one column per
  // step, so every register index is static while the column loop stays a runtime loop
  double w[RPT][RJB];
  int grow[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int i = threadIdx.x + q * PNT;
    grow[q] = i < nloc ? r0 + i : NONE;
#pragma unroll
    for (int c = 0; c < RJB; ++c) w[q][c] = (i < nloc && c < jb) ? W[(long long)(a.j0 + c) * ld + r0 + i] : 0.0;
  }
  for (int j = 0; j < jb; ++j) {
    const int rj = a.j0 + j;
    const int nrem = jb - j - 1;  // remaining columns: window slots 1..nrem
    // ---- norm of the column below the diagonal, and its diagonal entry
    double pn = 0.0, ap = 0.0;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (grow[q] != NONE && grow[q] > rj) pn = fma(w[q][0], w[q][0], pn);
      if (grow[q] == rj) ap = w[q][0];
    }
    pn = warp_sum(pn);
    ap = warp_sum(ap);
    if (lane == 0) {
      red2[warp] = pn;
      red2[NWW + warp] = ap;
    }
    __syncthreads();
    if ((int)threadIdx.x < G) {  // push this CTA's sums into every CTA's inbox
      double x = 0.0, y = 0.0;
#pragma unroll
      for (int k = 0; k < NWW; ++k) {
        x += red2[k];
        y += red2[NWW + k];
      }
      double* dst = cl.map_shared_rank(&nin[0][0], (int)threadIdx.x);
      dst[2 * rank] = x;
      dst[2 * rank + 1] = y;
    }
    cl.sync();
    double xnorm2 = 0.0, alpha = 0.0;
    for (int r = 0; r < G; ++r) {  // rank order: identical in every CTA
      xnorm2 += nin[r][0];
      alpha += nin[r][1];
    }
    double tau = 0.0, beta = alpha, scal = 1.0;
    if (xnorm2 > 0.0) {  // dlarfg
      beta = -copysign(hypot(alpha, sqrt(xnorm2)), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (rank == 0 && threadIdx.x == 0) a.tau[rj] = tau;
    double v[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (grow[q] != NONE && grow[q] > rj) {
        w[q][0] *= scal;
        v[q] = w[q][0];
      } else {
        v[q] = grow[q] == rj ? 1.0 : 0.0;
      }
    }
    const bool upd = tau != 0.0 && nrem > 0;  // uniform over the cluster
    if (upd) {
      // ---- partial dots d_c = sum_rows v w[:, c], c = 1..nrem, reduced within each warp
#pragma unroll
      for (int c8 = 0; c8 < RJB; c8 += 8) {
        if (c8 > nrem) break;
        double vals[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          vals[k] = 0.0;
#pragma unroll
          for (int q = 0; q < RPT; ++q) vals[k] = fma(v[q], w[q][c8 + k], vals[k]);
        }
#pragma unroll
        for (int st = 4; st >= 1; st >>= 1) {
          const bool up = (lane & st) != 0;
#pragma unroll
          for (int k = 0; k < st; ++k) {
            const double send = up ? vals[k] : vals[k + st];
            const double keep = up ? vals[k + st] : vals[k];
            vals[k] = keep + __shfl_xor_sync(0xffffffffu, send, st);
          }
        }
        vals[0] += __shfl_xor_sync(0xffffffffu, vals[0], 8);
        vals[0] += __shfl_xor_sync(0xffffffffu, vals[0], 16);
        if (lane < 8) wsum[warp][c8 + lane] = vals[0];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < G * RJB; e += PNT) {  // CTA partials -> every CTA's inbox
        const int col = e % RJB, dest = e / RJB;
        if (col >= 1 && col <= nrem) {
          double d = 0.0;
#pragma unroll
          for (int k = 0; k < NWW; ++k) d += wsum[k][col];
          cl.map_shared_rank(&din[0][0], dest)[rank * RJB + col] = d;
        }
      }
    }
    cl.sync();
    if (upd) {
      if ((int)threadIdx.x < RJB) {
        double d = 0.0;
        for (int r = 0; r < G; ++r) d += din[r][threadIdx.x];
        sw[threadIdx.x] = d * tau;
      }
      __syncthreads();
#pragma unroll
      for (int c = 1; c < RJB; ++c) {
        const double wc = c <= nrem ? sw[c] : 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) w[q][c] = fma(-wc, v[q], w[q][c]);
      }
    }
    // ---- column j is final: R above the diagonal, beta on it, the reflector below
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      if (grow[q] == NONE) continue;
      const int i = threadIdx.x + q * PNT;
      const double val = grow[q] == rj ? beta : w[q][0];
      W[(long long)rj * ld + r0 + i] = val;
      if (a.T) P[j * ldp + i] = val;
    }
    // ---- shift the register window
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
#pragma unroll
      for (int c = 0; c + 1 < RJB; ++c) w[q][c] = w[q][c + 1];
      w[q][RJB - 1] = 0.0;
    }
  }
  if (a.T == nullptr) {
    cl.sync();
    return;
  }
  panel_emit_vt<PNT>(a, P, ldp, nloc, r0, cl);
}

constexpr int CLUSTER_SMEM_DOUBLES = 25 * 1024;  // 200 KB of panel rows per CTA

// Launch the cluster panel when the panel fits 16 CTAs' shared memory; false otherwise.
bool launch_panel_cluster(const PanelArgs& pa, int mrows, int jb, cudaStream_t s) {
  static PerDevice<int> ok_dev(-1);
  int& ok = ok_dev();
  static const int disabled = std::getenv("QTT_PANEL_CLUSTER") && std::atoi(std::getenv("QTT_PANEL_CLUSTER")) == 0;
  if (disabled) return false;
  constexpr int CL = 16;
  const int chunk = (mrows + CL - 1) / CL;
  if ((long long)(chunk | 1) * jb > CLUSTER_SMEM_DOUBLES) return false;
  const size_t dyn = std::max<size_t>((size_t)(chunk | 1) * jb, pa.T ? 3 * NB * (NB + 1) : 0) * 8;
  if (ok < 0) {
    ok = cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                 cudaSuccess &&
             cudaFuncSetAttribute(panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  CLUSTER_SMEM_DOUBLES * 8) == cudaSuccess
         ? 1
         : 0;
    cudaGetLastError();
  }
  if (!ok) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(PNT);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, panel_cluster_kernel, pa);
  if (e != cudaSuccess) {  // e.g. 16-CTA clusters not schedulable at this size: fall back
    cudaGetLastError();
    if (std::getenv("QTT_DEBUG"))
      std::fprintf(stderr, "[qtt] cluster panel %dx%d not launched: %s\n", mrows, jb, cudaGetErrorString(e));
    return false;
  }
  QTT_CHECK_LAUNCH();
  return true;
}

// Launch the register-resident panel (16-CTA cluster) when jb <= 32 and each CTA's rows fit
// 3 per thread; false otherwise.
template <int RPT>
bool launch_panel_reg_t(const PanelArgs& pa, size_t dyn, cudaStream_t s) {
  static PerDevice<int> ok_dev(-1);
  int& ok = ok_dev();
  if (ok < 0) {
    ok = cudaFuncSetAttribute(panel_reg_kernel<RPT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                 cudaSuccess &&
             cudaFuncSetAttribute(panel_reg_kernel<RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  CLUSTER_SMEM_DOUBLES * 8) == cudaSuccess
         ? 1
         : 0;
    cudaGetLastError();
  }
  if (!ok) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(PNT);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, panel_reg_kernel<RPT>, pa);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  QTT_CHECK_LAUNCH();
  return true;
}

bool launch_panel_reg(const PanelArgs& pa, int mrows, int jb, cudaStream_t s) {
  static const int disabled = std::getenv("QTT_PANEL_REG") && std::atoi(std::getenv("QTT_PANEL_REG")) == 0;
  if (disabled || jb > RJB) return false;
  const int chunk = (mrows + 15) / 16;
  const int rpt = (chunk + PNT - 1) / PNT;
  if (rpt > 3) return false;
  const size_t dyn = std::max<size_t>(pa.T ? (size_t)(chunk | 1) * jb : 0, pa.T ? 3 * NB * (NB + 1) : 0) * 8;
  if (dyn > (size_t)CLUSTER_SMEM_DOUBLES * 8) return false;
  switch (rpt) {
    case 1: return launch_panel_reg_t<1>(pa, dyn, s);
    case 2: return launch_panel_reg_t<2>(pa, dyn, s);
    default: return launch_panel_reg_t<3>(pa, dyn, s);
  }
}

int panel_grid(int rows) {
  // enough CTAs that each owns >= ~256 rows, capped at one wave
  return std::max(1, std::min(128, (rows + 255) / 256));
}

// CTAs for the shared-memory panel: each row block must fit SMEM_PANEL_DOUBLES.
// Small row blocks (~QTT_PANEL_ROWS rows, default 64) keep the per-column work of
// each CTA short: the panel is latency-bound, so more CTAs beat fuller ones.
int panel_smem_grid(int rows, int jb) {
  static const int target = std::getenv("QTT_PANEL_ROWS") ? std::atoi(std::getenv("QTT_PANEL_ROWS")) : 64;
  const int max_rows = SMEM_PANEL_DOUBLES / std::max(1, jb) - 1;  // (odd pitch: chunk | 1)
  const int need = std::max(1, (rows + max_rows - 1) / max_rows);
  const int want = std::min(148, std::max(1, (rows + target - 1) / std::max(1, target)));
  return std::max(need, want);
}

}  // namespace

// QTT_DEBUG: per-stage CUDA-event timing of the blocked QR, printed per call.
struct QrTimer {
  bool on;
  cudaStream_t s;
  std::vector<cudaEvent_t> ev;
  std::vector<int> stage;
  double ms[6] = {0, 0, 0, 0, 0, 0};
  explicit QrTimer(cudaStream_t st) : on(std::getenv("QTT_DEBUG") != nullptr), s(st) {}
  void mark(int st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
    stage.push_back(st);
  }
  void report(int m, int n) {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back());
    for (size_t i = 1; i < ev.size(); ++i) {
      float t = 0;
      cudaEventElapsedTime(&t, ev[i - 1], ev[i]);
      ms[stage[i]] += t;
    }
    for (auto e : ev) cudaEventDestroy(e);
    std::fprintf(stderr, "[qtt] geqrf %dx%d ms: panel %.2f v+gram+T %.2f Y1 %.2f Y2 %.2f update %.2f\n", m, n,
                 ms[1], ms[2], ms[3], ms[4], ms[5]);
  }
};

// Two-level blocked Householder QR: 64-column panels (panel_smem_kernel) are applied
// to the rest of their 256-column outer block one at a time, while the columns right
// of the outer block get ONE compact-WY update per outer block (V_big: m x 256,
// T_big assembled from the panel T's), so the large trailing matrix is streamed
// through HBM a quarter as often and its GEMMs run with K = 256.
namespace {
constexpr int NB2 = 256;

void apply_wy_left(Ctx& c, const double* V, int mrows, int jb, const double* T, long long ldt, double* C,
                   long long ld, int n2, DBuf& Y1, DBuf& Y2, DBuf& Wsk, bool trans_t = true) {
  // C (mrows x n2, column-major ld) <- (I - V T V^T)^T C = C - V T^T (V^T C)   (trans_t)
  //                                 <- (I - V T V^T) C   = C - V T (V^T C)     (!trans_t, dorgqr)
  if (Y1.n < (long long)jb * n2) Y1.alloc((long long)jb * n2, c.stream);
  if (Y2.n < (long long)jb * n2) Y2.alloc((long long)jb * n2, c.stream);
  {  // Y1 = V^T C   (jb x n2)
    GemmArgs g;
    g.M = jb; g.N = n2; g.K = mrows;
    g.A = V; g.a_rs = mrows; g.a_cs = 1;
    g.B = C; g.b_rs = 1; g.b_cs = ld;
    gemm_set_C(g, Y1.p, n2);
    const long long need = gemm_workspace_hint(g);
    if (Wsk.n < need) Wsk.alloc(need, c.stream);
    gemm(g, c.stream, Wsk.p, Wsk.n);
  }
  {  // Y2 = T^T Y1
    GemmArgs g;
    g.M = jb; g.N = n2; g.K = jb;
    g.A = T;
    g.a_rs = trans_t ? 1 : ldt;
    g.a_cs = trans_t ? ldt : 1;
    gemm_set_B(g, Y1.p, n2, false);
    gemm_set_C(g, Y2.p, n2);
    gemm(g, c.stream);
  }
  {  // C -= V Y2
    GemmArgs g;
    g.M = mrows; g.N = n2; g.K = jb;
    g.A = V; g.a_rs = 1; g.a_cs = mrows;
    gemm_set_B(g, Y2.p, n2, false);
    g.C = C; g.c_rs = 1; g.c_cs = ld;
    g.alpha = -1.0; g.beta = 1.0;
    gemm(g, c.stream);
  }
}

// The outer compact-WY update in the transposed orientation, so both big products read
// K-contiguous operands and take the TMA GEMM path (gemm_tma.cu):
//   Y1^T = C^T V            (n2 x jb;  A = C^T = C's column-major storage, B = V^T stored [jb][mrows])
//   Y2^T = Y1^T T           (small)
//   C^T -= Y2^T V^T         (A = Y2^T [n2][jb], B = VT [mrows][jb], the row-major copy of V)
// C is column-major (ld), i.e. C^T row-major with leading dimension ld: same storage, no copy.
void apply_wy_left_t(Ctx& c, const double* V, int mrows, int jb, const double* T, long long ldt, double* C,
                     long long ld, int n2, DBuf& Y1, DBuf& Y2, DBuf& Wsk, DBuf& VT) {
  if (Y1.n < (long long)jb * n2) Y1.alloc((long long)jb * n2, c.stream);
  if (Y2.n < (long long)jb * n2) Y2.alloc((long long)jb * n2, c.stream);
  if (VT.n < (long long)mrows * jb) VT.alloc((long long)mrows * jb, c.stream);
  transpose_rows(V, VT.p, jb, mrows, jb, c.stream);  // V as [jb][mrows] -> VT [mrows][jb]
  {  // Y1T [n2][jb] = C^T V
    GemmArgs g;
    g.M = n2; g.N = jb; g.K = mrows;
    g.A = C; g.a_rs = ld; g.a_cs = 1;
    g.B = V; g.b_rs = 1; g.b_cs = mrows;
    gemm_set_C(g, Y1.p, jb);
    const long long need = gemm_workspace_hint(g);
    if (Wsk.n < need) Wsk.alloc(need, c.stream);
    gemm(g, c.stream, Wsk.p, Wsk.n);
  }
  {  // Y2T [n2][jb] = Y1T T   (Y2 = T^T Y1)
    GemmArgs g;
    g.M = n2; g.N = jb; g.K = jb;
    gemm_set_A(g, Y1.p, jb, false);
    g.B = T; g.b_rs = ldt; g.b_cs = 1;
    gemm_set_C(g, Y2.p, jb);
    gemm(g, c.stream);
  }
  {  // C^T [n2][mrows] -= Y2T VT^T
    GemmArgs g;
    g.M = n2; g.N = mrows; g.K = jb;
    gemm_set_A(g, Y2.p, jb, false);
    g.B = VT.p; g.b_rs = 1; g.b_cs = jb;
    g.C = C; g.c_rs = ld; g.c_cs = 1;
    g.alpha = -1.0; g.beta = 1.0;
    const long long need = gemm_workspace_hint(g);
    if (Wsk.n < need) Wsk.alloc(need, c.stream);
    gemm(g, c.stream, Wsk.p, Wsk.n);
  }
}

void gram_vtv(Ctx& c, const double* V, int mrows, int jb, double* G, DBuf& Wsk) {  // G = V^T V (jb x jb)
  GemmArgs g;
  g.M = jb; g.N = jb; g.K = mrows;
  g.A = V; g.a_rs = mrows; g.a_cs = 1;
  g.B = V; g.b_rs = 1; g.b_cs = mrows;
  gemm_set_C(g, G, jb);
  const long long need = gemm_workspace_hint(g);
  if (Wsk.n < need) Wsk.alloc(need, c.stream);
  gemm(g, c.stream, Wsk.p, Wsk.n);
}

__global__ void copy_block_kernel(const double* src, int rows, int cols, long long lds, double* dst, long long ldd) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int i = e / cols, j = e % cols;
    dst[i * ldd + j] = src[i * lds + j];
  }
}

}  // namespace

void geqrf_blocked(Ctx& c, double* W, int m, int n, double* tau) {
  const int k = std::min(m, n);
  QrTimer tm(c.stream);
  tm.mark(0);
  static const bool tl_on = std::getenv("QTT_DEBUG") && std::atoi(std::getenv("QTT_DEBUG")) >= 2;
  DBuf tlbuf;
  if (tl_on) {
    tlbuf.alloc(8, c.stream);
    QTT_CUDA(cudaMemsetAsync(tlbuf.p, 0, 64, c.stream));
  }
  DBuf red(149LL * (NB + 2), c.stream), Vb((long long)m * NB, c.stream), Gram(NB * NB, c.stream),
      T(NB * NB, c.stream), Y1, Y2, Wsk;
  DBuf Vbig, Gbig, Tbig, P1, VTbig;
  const long long ld = m;
  for (int J0 = 0; J0 < k; J0 += NB2) {
    const int JB = std::min(NB2, k - J0);
    const int jend = J0 + JB;  // columns right of this are updated once per outer block
    const bool outer = n - jend > 0 && JB > NB / 2;
    if (outer) {
      Tbig.alloc((long long)JB * JB, c.stream);
      QTT_CUDA(cudaMemsetAsync(Tbig.p, 0, (size_t)JB * JB * 8, c.stream));
    }
    // panel width: 64, or 32 when a 64-wide panel would not fit one 16-CTA cluster
    static const int cl_rows = 16 * (CLUSTER_SMEM_DOUBLES / NB);
    static const bool reg_on = !(std::getenv("QTT_PANEL_REG") && std::atoi(std::getenv("QTT_PANEL_REG")) == 0);
    const bool reg_fits = reg_on && (m - J0 + 15) / 16 <= 3 * PNT;  // register panel: 32 columns
    const int pw = (reg_fits || m - J0 > cl_rows) ? NB / 2 : NB;
    for (int j0 = J0; j0 < jend; j0 += pw) {
      const int jb = std::min(pw, jend - j0);
      const int mrows = m - j0;
      const int n2 = (outer ? jend : n) - j0 - jb;
      const bool need_t = n2 > 0 || outer;
      PanelArgs pa{W, ld, m, j0, jb, tau, red.p, tlbuf.p ? (unsigned long long*)tlbuf.p : nullptr};
      if (need_t) {  // the cluster panel also emits V and T (and T's diagonal block of T_big)
        pa.Vb = Vb.p;
        pa.T = T.p;
        pa.Tb = outer ? Tbig.p : nullptr;
        pa.ldtb = JB;
        pa.tb_off = j0 - J0;
      }
      const int Gs = panel_smem_grid(mrows, jb);
      bool have_vt = false;
      if (launch_panel_reg(pa, mrows, jb, c.stream) || launch_panel_cluster(pa, mrows, jb, c.stream)) {
        have_vt = need_t;
      } else if (Gs <= 148) {
        static PerDevice<bool> attr_dev(false);
        bool& attr = attr_dev();
        if (!attr) {
          QTT_CUDA(cudaFuncSetAttribute(panel_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        SMEM_PANEL_DOUBLES * 8));
          attr = true;
        }
        const int chunk = (mrows + Gs - 1) / Gs;
        void* args[] = {(void*)&pa};
        QTT_CUDA(cudaLaunchCooperativeKernel((void*)panel_smem_kernel, dim3(Gs), dim3(PNT), args,
                                             (size_t)(chunk | 1) * jb * 8, c.stream));
      } else {
        const int G = panel_grid(mrows);
        void* args[] = {(void*)&pa};
        QTT_CUDA(cudaLaunchCooperativeKernel((void*)panel_kernel, dim3(G), dim3(PNT), args, 0, c.stream));
      }
      QTT_CHECK_LAUNCH();
      tm.mark(1);
      // inner update: the rest of the outer block (or of the matrix when there is no outer step)
      if (!need_t) continue;
      if (!have_vt) {
      build_v_kernel<<<std::min(1184, cdiv((long long)mrows * jb, 256)), 256, 0, c.stream>>>(W, ld, j0, mrows,
                                                                                            jb, Vb.p);
      QTT_CHECK_LAUNCH();
      gram_vtv(c, Vb.p, mrows, jb, Gram.p, Wsk);
      build_t_kernel<<<1, NB, 0, c.stream>>>(Gram.p, tau + j0, jb, T.p);
      QTT_CHECK_LAUNCH();
      if (outer) {  // keep the panel T as a diagonal block of T_big
        copy_block_kernel<<<16, 256, 0, c.stream>>>(T.p, jb, jb, jb, Tbig.p + (long long)(j0 - J0) * JB + (j0 - J0),
                                                    JB);
        QTT_CHECK_LAUNCH();
      }
      }
      tm.mark(2);
      if (n2 > 0)
        apply_wy_left(c, Vb.p, mrows, jb, T.p, jb, W + (long long)(j0 + jb) * ld + j0, ld, n2, Y1, Y2, Wsk);
      tm.mark(5);
    }
    if (!outer) continue;
    // ---- one compact-WY update of the columns right of the outer block
    const int mrowsJ = m - J0;
    const int n2 = n - jend;
    Vbig.alloc((long long)mrowsJ * JB, c.stream);
    build_v_kernel<<<std::min(1184, cdiv((long long)mrowsJ * JB, 256)), 256, 0, c.stream>>>(W, ld, J0, mrowsJ, JB,
                                                                                           Vbig.p);
    QTT_CHECK_LAUNCH();
    Gbig.alloc((long long)JB * JB, c.stream);
    gram_vtv(c, Vbig.p, mrowsJ, JB, Gbig.p, Wsk);
    // T_big = [[T_1:k, -T_1:k (V_1:k^T V_k+1) T_k+1], [0, T_k+1]]  (dlarft block recursion)
    P1.alloc((long long)JB * NB, c.stream);
    for (int c0 = pw; c0 < JB; c0 += pw) {
      const int w = std::min(pw, JB - c0);
      {  // P1 (c0 x w) = T_big[0:c0, 0:c0] @ Gram[0:c0, c0:c0+w]
        GemmArgs g;
        g.M = c0; g.N = w; g.K = c0;
        gemm_set_A(g, Tbig.p, JB, false);
        gemm_set_B(g, Gbig.p + c0, JB, false);
        gemm_set_C(g, P1.p, w);
        gemm(g, c.stream);
      }
      {  // T_big[0:c0, c0:c0+w] = -P1 @ T_big[c0:c0+w, c0:c0+w]
        GemmArgs g;
        g.M = c0; g.N = w; g.K = w;
        gemm_set_A(g, P1.p, w, false);
        gemm_set_B(g, Tbig.p + (long long)c0 * JB + c0, JB, false);
        gemm_set_C(g, Tbig.p + c0, JB);
        g.alpha = -1.0;
        gemm(g, c.stream);
      }
    }
    tm.mark(2);
    apply_wy_left_t(c, Vbig.p, mrowsJ, JB, Tbig.p, JB, W + (long long)jend * ld + J0, ld, n2, Y1, Y2, Wsk, VTbig);
    tm.mark(5);
  }
  tm.report(m, n);
  if (tlbuf.p) {
    unsigned long long h[5];
    QTT_CUDA(cudaMemcpyAsync(h, tlbuf.p, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    QTT_CUDA(cudaStreamSynchronize(c.stream));
    const double cols = std::max(1, std::min(m, n));
    std::fprintf(stderr, "[qtt] geqrf %dx%d panel CTA0 ns/column: norm %.0f bar1 %.0f dlarfg+dots %.0f bar2 %.0f "
                 "reduce+update %.0f\n", m, n, h[0] / cols, h[1] / cols, h[2] / cols, h[3] / cols, h[4] / cols);
  }
}

namespace {
__global__ void eye_kernel(double* Q, int m, int k) {  // column-major m x k identity
  const long long total = (long long)m * k;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    Q[e] = (e % m) == (e / m) ? 1.0 : 0.0;
}
}  // namespace

// dorgqr, blocked: Q = H_1 ... H_k I[:, :k], panels applied last to first, each as one
// compact-WY product C <- (I - V T V^T) C on the trailing block Q[j0:, j0:].
void orgqr_blocked(Ctx& c, const double* W, int m, int k, const double* tau, double* Q) {
  eye_kernel<<<(int)std::min<long long>(cdiv((long long)m * k, 256), 1184), 256, 0, c.stream>>>(Q, m, k);
  QTT_CHECK_LAUNCH();
  DBuf Vb((long long)m * NB, c.stream), Gram(NB * NB, c.stream), T(NB * NB, c.stream), Y1, Y2, Wsk;
  for (int j0 = ((k - 1) / NB) * NB; j0 >= 0; j0 -= NB) {
    const int jb = std::min(NB, k - j0);
    const int mrows = m - j0;
    build_v_kernel<<<std::min(1184, cdiv((long long)mrows * jb, 256)), 256, 0, c.stream>>>(W, m, j0, mrows, jb,
                                                                                          Vb.p);
    QTT_CHECK_LAUNCH();
    gram_vtv(c, Vb.p, mrows, jb, Gram.p, Wsk);
    build_t_kernel<<<1, NB, 0, c.stream>>>(Gram.p, tau + j0, jb, T.p);
    QTT_CHECK_LAUNCH();
    apply_wy_left(c, Vb.p, mrows, jb, T.p, jb, Q + (long long)j0 * m + j0, m, k - j0, Y1, Y2, Wsk, false);
  }
}

}  // namespace qtt
