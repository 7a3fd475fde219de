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
};

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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* W = a.W;
  const long long ld = a.ld;
  for (int e = threadIdx.x; e < nloc * a.jb; e += PNT) {
    const int c = e / nloc, i = e % nloc;
    P[e] = W[(long long)(a.j0 + c) * ld + r0 + i];
  }
  __syncthreads();
  for (int j = 0; j < a.jb; ++j) {
    const int rj = a.j0 + j;
    double* v = P + j * nloc;  // local rows r0..r1
    const int ib = max(0, rj + 1 - r0);  // first local row strictly below rj
    double part = 0.0;
    for (int i = ib + threadIdx.x; i < nloc; i += PNT) part += v[i] * v[i];
    part = block_sum(part, red);
    const bool own_rj = (rj >= r0 && rj < r1);
    if (threadIdx.x == 0) {
      a.red[blockIdx.x * (NB + 2)] = part;
      a.red[blockIdx.x * (NB + 2) + NB + 1] = own_rj ? v[rj - r0] : 0.0;  // alpha
    }
    cg::this_grid().sync();
    double xn = 0.0, al = 0.0;
    for (int b = threadIdx.x; b < G; b += PNT) {
      xn += __ldcg(a.red + b * (NB + 2));
      al += __ldcg(a.red + b * (NB + 2) + NB + 1);
    }
    const double xnorm2 = block_sum(xn, red);
    const double alpha = block_sum(al, red);  // exactly one CTA contributed
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
    if (t != 0.0 && nrem > 0) {
      for (int cc = warp; cc < nrem; cc += PNT / 32) {
        const double* wc = P + (j + 1 + cc) * nloc;
        double s = 0.0;
        for (int i = ib + lane; i < nloc; i += 32) s += v[i] * wc[i];
        s = warp_sum(s);
        if (lane == 0) a.red[blockIdx.x * (NB + 2) + 1 + cc] = s + (own_rj ? wc[rj - r0] : 0.0);
      }
    }
    cg::this_grid().sync();
    if (t != 0.0 && nrem > 0) {
      {  // 4 threads per column, all partial loads in flight at once; fixed order
        const int cc = threadIdx.x >> 2, sub = threadIdx.x & 3;
        double s = 0.0;
        if (cc < nrem)
          for (int b = sub; b < G; b += 4) s += __ldcg(a.red + b * (NB + 2) + 1 + cc);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (sub == 0 && cc < nrem) sw[cc] = s * t;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < nrem * nloc; e += PNT) {
        const int cc = e / nloc, i = e % nloc;
        double* wc = P + (j + 1 + cc) * nloc;
        if (i >= ib) wc[i] -= sw[cc] * v[i];
        else if (own_rj && i == rj - r0) wc[i] -= sw[cc];
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < a.jb; j += PNT) {
    const int rj = a.j0 + j;
    if (rj >= r0 && rj < r1) P[j * nloc + (rj - r0)] = sbeta[j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nloc * a.jb; e += PNT) {
    const int c = e / nloc, i = e % nloc;
    W[(long long)(a.j0 + c) * ld + r0 + i] = P[e];
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
  const int max_rows = SMEM_PANEL_DOUBLES / std::max(1, jb);
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

void geqrf_blocked(Ctx& c, double* W, int m, int n, double* tau) {
  const int k = std::min(m, n);
  QrTimer tm(c.stream);
  tm.mark(0);
  DBuf red(149LL * (NB + 2), c.stream), Vb((long long)m * NB, c.stream), Gram(NB * NB, c.stream),
      T(NB * NB, c.stream), Y1, Y2, Wsk;
  const long long ld = m;
  for (int j0 = 0; j0 < k; j0 += NB) {
    const int jb = std::min(NB, k - j0);
    const int mrows = m - j0;
    PanelArgs pa{W, ld, m, j0, jb, tau, red.p};
    const int Gs = panel_smem_grid(mrows, jb);
    if (Gs <= 148) {
      static bool attr = false;
      if (!attr) {
        QTT_CUDA(cudaFuncSetAttribute(panel_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_PANEL_DOUBLES * 8));
        attr = true;
      }
      const int chunk = (mrows + Gs - 1) / Gs;
      void* args[] = {(void*)&pa};
      QTT_CUDA(cudaLaunchCooperativeKernel((void*)panel_smem_kernel, dim3(Gs), dim3(PNT), args,
                                           (size_t)chunk * jb * 8, c.stream));
    } else {
      const int G = panel_grid(mrows);
      void* args[] = {(void*)&pa};
      QTT_CUDA(cudaLaunchCooperativeKernel((void*)panel_kernel, dim3(G), dim3(PNT), args, 0, c.stream));
    }
    QTT_CHECK_LAUNCH();
    tm.mark(1);
    const int n2 = n - j0 - jb;
    if (n2 <= 0) continue;
    build_v_kernel<<<std::min(1184, cdiv((long long)mrows * jb, 256)), 256, 0, c.stream>>>(W, ld, j0, mrows,
                                                                                          jb, Vb.p);
    QTT_CHECK_LAUNCH();
    {  // Gram = Vb^T Vb
      GemmArgs g;
      g.M = jb; g.N = jb; g.K = mrows;
      g.A = Vb.p; g.a_rs = mrows; g.a_cs = 1;
      g.B = Vb.p; g.b_rs = 1; g.b_cs = mrows;
      gemm_set_C(g, Gram.p, jb);
      const long long need = gemm_workspace_hint(g);  // one output tile, K = mrows: split K
      if (Wsk.n < need) Wsk.alloc(need, c.stream);
      gemm(g, c.stream, Wsk.p, Wsk.n);
    }
    build_t_kernel<<<1, NB, 0, c.stream>>>(Gram.p, tau + j0, jb, T.p);
    QTT_CHECK_LAUNCH();
    tm.mark(2);
    if (Y1.n < (long long)jb * n2) Y1.alloc((long long)jb * n2, c.stream);
    if (Y2.n < (long long)jb * n2) Y2.alloc((long long)jb * n2, c.stream);
    double* C = W + (long long)(j0 + jb) * ld + j0;
    {  // Y1 = Vb^T C   (jb x n2)
      GemmArgs g;
      g.M = jb; g.N = n2; g.K = mrows;
      g.A = Vb.p; g.a_rs = mrows; g.a_cs = 1;
      g.B = C; g.b_rs = 1; g.b_cs = ld;
      gemm_set_C(g, Y1.p, n2);
      const long long need = gemm_workspace_hint(g);
      if (Wsk.n < need) Wsk.alloc(need, c.stream);
      gemm(g, c.stream, Wsk.p, Wsk.n);
    }
    tm.mark(3);
    {  // Y2 = T^T Y1
      GemmArgs g;
      g.M = jb; g.N = n2; g.K = jb;
      g.A = T.p; g.a_rs = 1; g.a_cs = jb;
      gemm_set_B(g, Y1.p, n2, false);
      gemm_set_C(g, Y2.p, n2);
      gemm(g, c.stream);
    }
    tm.mark(4);
    {  // C -= Vb Y2
      GemmArgs g;
      g.M = mrows; g.N = n2; g.K = jb;
      g.A = Vb.p; g.a_rs = 1; g.a_cs = mrows;
      gemm_set_B(g, Y2.p, n2, false);
      g.C = C; g.c_rs = 1; g.c_cs = ld;
      g.alpha = -1.0; g.beta = 1.0;
      gemm(g, c.stream);
    }
    tm.mark(5);
  }
  tm.report(m, n);
}

}  // namespace qtt
