// Device AMEn sweep and driver (amen.py:163-510), orchestrated from C++ on the
// context stream.  Host round trips happen only where the reference makes a
// data-dependent decision: SVD rank choice, Cholesky pivot check, CG stopping
// (polled in chunks), the per-sweep estimate and the certification.
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "amen.cuh"
#include "cg_fused.cuh"
#include "cg_tma.cuh"
#include "tma_tile.cuh"
#include "chol_fused.cuh"
#include "contract.cuh"
#include "gemm.cuh"
#include "linalg.cuh"

namespace qtt {

const double* DrawStream::take(long long k) {
  if (pos + k > n) throw Error(QTT_ERR_ARG, "random draw stream exhausted");
  const double* out = p + pos;
  pos += k;
  return out;
}

namespace {


// ------------------------------------------------------------------ CG kernels
// Device state in Ctx::scal: [0] rho [1] alpha [2] rnorm [3] beta
// Ctx::flags: [0] done [1] iterations
constexpr int RB = 148;  // reduction blocks

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// two simultaneous block sums (256 threads)
__device__ void block_sum2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = wsum(a);
  b = wsum(b);
  __syncthreads();
  if (lane == 0) { red[warp] = a; red[8 + warp] = b; }
  __syncthreads();
  if (warp == 0) {
    double x = lane < 8 ? red[lane] : 0.0, y = lane < 8 ? red[8 + lane] : 0.0;
    x = wsum(x);
    y = wsum(y);
    if (lane == 0) { red[16] = x; red[17] = y; }
  }
  __syncthreads();
  a = red[16];
  b = red[17];
}

// r0: residual;  computes z = invd*r, p = z, rho = r.z, rnorm = |r|; done if rnorm < atol.
__global__ void __launch_bounds__(256) cg_start_kernel(const double* r, const double* invd, double* z,
                                                       double* p, long long n, double atol, double* part,
                                                       unsigned* counter, double* scal, int* flags) {
  __shared__ double red[20];
  __shared__ bool last;
  double rr = 0, rz = 0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const double ri = r[i], zi = ri * invd[i];
    z[i] = zi;
    p[i] = zi;
    rr += ri * ri;
    rz += ri * zi;
  }
  block_sum2(rr, rz, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = rr;
    part[2 * blockIdx.x + 1] = rz;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a = 0, b = 0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += 256) {
    a += ((volatile double*)part)[2 * i];
    b += ((volatile double*)part)[2 * i + 1];
  }
  block_sum2(a, b, red);
  if (threadIdx.x == 0) {
    *counter = 0u;
    const double rn = sqrt(a);
    scal[2] = rn;
    scal[0] = b;
    flags[1] = 0;
    flags[0] = (rn < atol) ? 1 : 0;
  }
}

// alpha = rho / (p.q)
__global__ void __launch_bounds__(256) cg_alpha_kernel(const double* p, const double* q, long long n,
                                                       double* part, unsigned* counter, double* scal,
                                                       const int* flags) {
  if (flags[0]) return;
  __shared__ double red[20];
  __shared__ bool last;
  double pq = 0, dummy = 0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    pq += p[i] * q[i];
  block_sum2(pq, dummy, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = pq;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a = 0, b = 0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += 256) a += ((volatile double*)part)[i];
  block_sum2(a, b, red);
  if (threadIdx.x == 0) {
    *counter = 0u;
    scal[1] = scal[0] / a;
  }
}

// x += alpha p; r -= alpha q; z = invd r; then rnorm, rho_new; stopping; beta.
__global__ void __launch_bounds__(256) cg_update_kernel(double* x, double* r, double* z, const double* p,
                                                        const double* q, const double* invd, long long n,
                                                        double atol, int maxiter, double* part,
                                                        unsigned* counter, double* scal, int* flags) {
  if (flags[0]) return;
  __shared__ double red[20];
  __shared__ bool last;
  const double alpha = scal[1];
  double rr = 0, rz = 0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    const double zi = ri * invd[i];
    z[i] = zi;
    rr += ri * ri;
    rz += ri * zi;
  }
  block_sum2(rr, rz, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = rr;
    part[2 * blockIdx.x + 1] = rz;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a = 0, b = 0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += 256) {
    a += ((volatile double*)part)[2 * i];
    b += ((volatile double*)part)[2 * i + 1];
  }
  block_sum2(a, b, red);
  if (threadIdx.x == 0) {
    *counter = 0u;
    const int it = flags[1] + 1;
    flags[1] = it;
    const double rn = sqrt(a);
    scal[2] = rn;
    if (rn < atol || it >= maxiter) {
      flags[0] = 1;
    } else {
      scal[3] = b / scal[0];
      scal[0] = b;
    }
  }
}

__global__ void cg_dir_kernel(double* p, const double* z, long long n, const double* scal,
                              const int* flags) {
  if (flags[0]) return;
  const double beta = scal[3];
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    p[i] = z[i] + beta * p[i];
}

// invd = 1 / (d > 0 ? d : 1)   (amen.py:197-199)
__global__ void jacobi_inv_kernel(const double* d, double* invd, long long n) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    invd[i] = 1.0 / (d[i] > 0 ? d[i] : 1.0);
}

__global__ void sum_abs_kernel(const double* a, long long n, double* out) {
  // non-negative doubles order like their bit patterns: integer atomicMax gives max|a|
  double m = 0.0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    m = fmax(m, fabs(a[i]));
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 16));
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 8));
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
  if ((threadIdx.x & 31) == 0 && m > 0)
    atomicMax((unsigned long long*)out, (unsigned long long)__double_as_longlong(m));
}

// Build aug = [U[:, :r] | E] where E is given as a strided view (rows x re).
__global__ void build_aug_kernel(const double* U, int ldu, int r, CMatView E, double* aug, int rows) {
  const int cols = r + E.cols;
  const long long total = (long long)rows * cols;
  for (long long e = blockIdx.x * 256LL + threadIdx.x; e < total; e += (long long)gridDim.x * 256) {
    const int i = (int)(e / cols), j = (int)(e % cols);
    aug[e] = j < r ? U[(long long)i * ldu + j] : E.p[i * E.rs + (j - r) * E.cs];
  }
}

inline int grid_for(long long n) {
  return (int)std::max<long long>(1, std::min<long long>(cdiv(n, 256), 1184));
}

// ------------------------------------------------------------------ helpers
struct Env {
  int b = 1, o = 1, k = 1;  // phi: (bra, op, ket); psi: (bra, rhs, 1)
  DBuf d;
};

Env unit_env(Ctx& c) {
  Env e;
  e.d.alloc(1, c.stream);
  fill(c, e.d.p, 1, 1.0);
  return e;
}



}  // namespace

DBuf solve_local_system(Ctx& c_, const LocalSystem& L, const double* rhs_p, const double* prev_p,
                        const AmenParams& prm_, int sweep_, int k, double& lam, int& iters,
                        bool profile) {
  const int m = L.m;
  const long long dim = (long long)L.lb * m * L.rb;
  DBuf mv_scratch;
  auto matvec = [&](const double* v, double* y, double alpha, double beta, const int* skip) {
    const long long need = local_matvec_scratch(L.lb, L.lo, L.lk, L.m, L.n, L.R1, L.rb, L.rk) +
                           (long long)L.lb * L.m * L.rb * 8;
    if (mv_scratch.n < need) mv_scratch.alloc(need, c_.stream);
    DBuf& sc = mv_scratch;
    local_matvec(L.phil, L.lb, L.lo, L.lk, L.Ap, L.m, L.n, L.R1, L.phir, L.rb, L.rk, v, y, alpha, beta,
                 {sc.p, sc.n}, c_.stream, skip);
  };
  iters = 0;
  DBuf u(dim, c_.stream);
  if (!prm_.local_iterative && dim <= prm_.direct_dim_cap) {
    // ---- direct: dense local matrix + Cholesky (amen.py:181-191)
    DBuf M(dim * dim, c_.stream);
    DBuf sc(local_dense_scratch(L.lb, L.lo, L.lk, L.m, L.n, L.R1), c_.stream);
    local_dense(L.phil, L.lb, L.lo, L.lk, L.A, L.m, L.n, L.R1, L.phir, L.rb, L.rk, M.p, {sc.p, sc.n},
                c_.stream);
    QTT_CUDA(cudaMemcpyAsync(u.p, rhs_p, dim * 8, cudaMemcpyDeviceToDevice, c_.stream));
    if (prm_.fused_cg) {  // one cooperative kernel: row sums + Cholesky + both solves
      QTT_CUDA(cudaMemsetAsync(c_.scal + 8, 0, 8, c_.stream));
      QTT_CUDA(cudaMemsetAsync(c_.flags + 3, 0, 4, c_.stream));
      DBuf Linv(chol_fused_linv_doubles((int)dim), c_.stream), ywork(dim, c_.stream);
      static const bool dbg = std::getenv("QTT_DEBUG") != nullptr;
      CholArgs ca{M.p, (int)dim, dim, u.p, c_.scal + 8, c_.flags + 3, Linv.p, ywork.p,
                  dbg ? (unsigned long long*)(c_.scal + 40) : nullptr};
      if (dbg) QTT_CUDA(cudaMemsetAsync(c_.scal + 40, 0, 6 * 8, c_.stream));
      chol_fused_launch(ca, chol_fused_grid(c_.device), c_.stream);
      if (dbg) {
        unsigned long long ph[6];
        QTT_CUDA(cudaMemcpyAsync(ph, c_.scal + 40, sizeof(ph), cudaMemcpyDeviceToHost, c_.stream));
        c_.sync();
        std::fprintf(stderr, "[qtt] chol dim %lld ns: rowsum %llu diag %llu panel %llu trail %llu inv %llu fwd %llu\n",
                     dim, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5]);
      }
      c_.stats.chol_solves++;
    } else {
      max_abs_row_sum(c_, M.p, (int)dim, dim, c_.scal + 8);
      potrf_lower(c_, M.p, (int)dim, dim, c_.flags + 3);
      potrs_lower(c_, M.p, (int)dim, dim, u.p);
    }
    double* pin = c_.host_scalars(2);
    QTT_CUDA(cudaMemcpyAsync(pin, c_.scal + 8, 8, cudaMemcpyDeviceToHost, c_.stream));
    QTT_CUDA(cudaMemcpyAsync(pin + 1, c_.flags + 3, 4, cudaMemcpyDeviceToHost, c_.stream));
    c_.sync();
    lam = pin[0];
    int info;
    std::memcpy(&info, pin + 1, 4);
    if (info != 0)
      throw Error(QTT_ERR_SOLVER, "local system not positive definite at sweep " + std::to_string(sweep_) +
                                      ", core " + std::to_string(k) + " (dim " + std::to_string(dim) +
                                      "): leading minor of order " + std::to_string(info) +
                                      " is not positive");
    return u;
  }
  // ---- iterative: Jacobi-PCG (amen.py:192-214, SciPy cg recurrence)
  c_.stats.cg_solves++;
  DBuf diag(dim, c_.stream), invd(dim, c_.stream);
  {
    DBuf sc((long long)L.lb * m * L.R1, c_.stream);
    local_diag(L.phil, L.lb, L.lo, L.A, m, L.R1, L.phir, L.rb, diag.p, {sc.p, sc.n}, c_.stream);
  }
  sum(c_, diag.p, dim, c_.scal + 8);  // lam = trace (before the non-positive replacement)
  jacobi_inv_kernel<<<grid_for(dim), 256, 0, c_.stream>>>(diag.p, invd.p, dim);
  QTT_CHECK_LAUNCH();
  nrm2(c_, rhs_p, dim, c_.scal + 9);
  QTT_CUDA(cudaMemsetAsync(c_.scal + 10, 0, 8, c_.stream));
  sum_abs_kernel<<<grid_for(dim), 256, 0, c_.stream>>>(prev_p, dim, c_.scal + 10);
  QTT_CHECK_LAUNCH();
  double h[3];
  read_scalars(c_, c_.scal + 8, 3, h);
  lam = h[0];
  const double bnorm = h[1];
  const bool xany = h[2] > 0;
  if (bnorm == 0.0) {  // scipy returns b itself
    QTT_CUDA(cudaMemcpyAsync(u.p, rhs_p, dim * 8, cudaMemcpyDeviceToDevice, c_.stream));
    return u;
  }
  const double rtol = std::max(0.05 * prm_.residual_tol, 1e-13);
  const double atol = rtol * bnorm;
  DBuf r(dim, c_.stream), z(dim, c_.stream), p(dim, c_.stream), q(dim, c_.stream);
  QTT_CUDA(cudaMemcpyAsync(u.p, prev_p, dim * 8, cudaMemcpyDeviceToDevice, c_.stream));
  QTT_CUDA(cudaMemcpyAsync(r.p, rhs_p, dim * 8, cudaMemcpyDeviceToDevice, c_.stream));
  const double kflops = local_matvec_flops(L.lb, L.lo, L.lk, L.m, L.n, L.R1, L.rb, L.rk);
  static const int tma_env = std::getenv("QTT_CG_TMA") ? std::atoi(std::getenv("QTT_CG_TMA")) : 1;
  if (prm_.fused_cg && tma_env != 0 && cg_tma_supported(L.lk, L.n) && L.lb == L.lk && L.rb == L.rk &&
      L.m == L.n) {
    // one persistent cooperative kernel on the TMA engine (cg_tma.cu); vectors transposed
    const int grid = cg_tma_grid(c_.device);
    const CGTmaPlan pl = cg_tma_plan(L.lb, L.m, L.R1, L.lk, L.n, L.rb, L.rk, grid);
    const long long K3 = (long long)L.R1 * L.rk, K3p = K3 + (K3 & 1);
    const long long rowsA = (long long)L.lk * L.n;  // (U,n)
    DBuf bT(dim, c_.stream), dT(dim, c_.stream), xT(dim, c_.stream);
    transpose_2d(rhs_p, bT.p, rowsA, L.rk, c_.stream);
    transpose_2d(invd.p, dT.p, rowsA, L.rk, c_.stream);
    transpose_2d(prev_p, xT.p, rowsA, L.rk, c_.stream);
    DBuf bop((long long)L.lb * L.m * L.R1 * rowsA, c_.stream);
    cg_fused_build_bop(L.phil, L.lb, L.lo, L.lk, L.Ap, L.m, L.n, L.R1, bop.p, c_.stream);
    DBuf phir_pad;
    const double* phir = L.phir;
    if (K3p != K3) {
      phir_pad.alloc((long long)L.rb * K3p, c_.stream);
      QTT_CUDA(cudaMemcpy2DAsync(phir_pad.p, K3p * 8, L.phir, K3 * 8, K3 * 8, L.rb, cudaMemcpyDeviceToDevice,
                                 c_.stream));
      phir = phir_pad.p;
    }
    DBuf t2((long long)L.lb * L.m * K3p, c_.stream), part3((long long)pl.S3 * dim, c_.stream);
    DBuf red(4LL * grid, c_.stream);
    CGTmaArgs a;
    std::memset(&a, 0, sizeof(a));
    make_tensor_map_2d(&a.map_bop, bop.p, (long long)L.lb * L.m * L.R1, rowsA, rowsA, pl.box1_a);
    make_tensor_map_2d(&a.map_z, z.p, L.rk, rowsA, rowsA, pl.box1_b);
    make_tensor_map_2d(&a.map_x, xT.p, L.rk, rowsA, rowsA, pl.box1_b);
    make_tensor_map_2d(&a.map_phir, phir, L.rb, K3, K3p, pl.box2_a);
    make_tensor_map_2d(&a.map_t2, t2.p, (long long)L.lb * L.m, K3, K3p, pl.box2_b);
    a.lb = L.lb; a.m = L.m; a.R1 = L.R1; a.lk = L.lk; a.n = L.n; a.rb = L.rb; a.rk = L.rk; a.K3p = K3p;
    a.p1_rb = pl.p1_rb; a.p1_cb = pl.p1_cb; a.p2_rb = pl.p2_rb; a.p2_cb = pl.p2_cb;
    a.p1_nf = pl.p1_nf; a.p1_dedupe = pl.p1_dedupe; a.p2_nf = pl.p2_nf; a.p2_dedupe = pl.p2_dedupe;
    a.box1_a = pl.box1_a; a.box1_b = pl.box1_b; a.box2_a = pl.box2_a; a.box2_b = pl.box2_b;
    a.stage_stride = pl.stage_stride;
    a.stages = pl.stages;
    a.p1_frun = pl.p1_frun;
    a.b = bT.p; a.invd = dT.p; a.x = xT.p; a.r = r.p; a.z = z.p; a.p = p.p; a.q = q.p;
    a.t2 = t2.p; a.part3 = part3.p; a.S3 = pl.S3; a.kt_per3 = pl.kt_per3; a.red = red.p;
    a.dim = dim; a.atol = atol; a.maxiter = prm_.local_iter_cap; a.xany = xany ? 1 : 0;
    a.out_iters = c_.flags + 8;
    a.out_rnorm = c_.scal + 20;
    a.out_mv_ns = (unsigned long long*)(c_.scal + 21);
    QTT_CUDA(cudaMemsetAsync(c_.scal + 21, 0, 8, c_.stream));
    static const bool dbg = std::getenv("QTT_DEBUG") != nullptr;
    a.phase_ns = dbg ? (unsigned long long*)(c_.scal + 32) : nullptr;
    if (dbg) QTT_CUDA(cudaMemsetAsync(c_.scal + 32, 0, 6 * 8, c_.stream));
    static const bool dbg2 = std::getenv("QTT_DEBUG") && std::atoi(std::getenv("QTT_DEBUG")) >= 2;
    DBuf ctans(dbg2 ? 3LL * grid + 8 : 1, c_.stream);
    if (dbg2) {
      QTT_CUDA(cudaMemsetAsync(ctans.p, 0, 24LL * grid + 64, c_.stream));
      a.cta_ns = (unsigned long long*)ctans.p;
    }
    cg_tma_launch(a, grid, c_.stream);
    if (dbg2) {
      std::vector<unsigned long long> h(3 * grid + 8);
      QTT_CUDA(cudaMemcpyAsync(h.data(), ctans.p, 24LL * grid + 64, cudaMemcpyDeviceToHost, c_.stream));
      c_.sync();
      int itd = 0;
      QTT_CUDA(cudaMemcpy(&itd, c_.flags + 8, 4, cudaMemcpyDeviceToHost));
      const double nmv = itd + (xany ? 1 : 0);
      std::fprintf(stderr, "[qtt] cg_tma CTA0 timeline us/matvec: p1 first-data %.2f loop-end %.2f epi-end %.2f "
                   "stream-end %.2f | p2 first-data %.2f loop-end %.2f epi-end %.2f stream-end %.2f\n",
                   h[3 * grid] / nmv / 1e3, h[3 * grid + 1] / nmv / 1e3, h[3 * grid + 2] / nmv / 1e3,
                   h[3 * grid + 3] / nmv / 1e3, h[3 * grid + 4] / nmv / 1e3, h[3 * grid + 5] / nmv / 1e3,
                   h[3 * grid + 6] / nmv / 1e3, h[3 * grid + 7] / nmv / 1e3);
      if (std::getenv("QTT_CTA_DUMP")) {
        std::fprintf(stderr, "[qtt] cta_dump");
        for (int i = 0; i < grid; ++i) std::fprintf(stderr, " %llu:%llu", h[2 * grid + i], h[i]);
        std::fprintf(stderr, "\n");
      }
      for (int ph = 0; ph < 2; ++ph) {
        std::vector<unsigned long long> v(h.begin() + ph * grid, h.begin() + (ph + 1) * grid);
        std::vector<unsigned long long> srt = v;
        std::sort(srt.begin(), srt.end());
        int amax = (int)(std::max_element(v.begin(), v.end()) - v.begin());
        std::fprintf(stderr, "[qtt] cg_tma phase%d per-CTA busy ns: min %llu med %llu p90 %llu max %llu (cta %d)\n",
                     ph + 1, srt[0], srt[grid / 2], srt[grid * 9 / 10], srt[grid - 1], amax);
      }
    }
    transpose_2d(xT.p, u.p, L.rk, rowsA, c_.stream);
    double* pin = c_.host_scalars(2);
    QTT_CUDA(cudaMemcpyAsync(pin, c_.scal + 21, 8, cudaMemcpyDeviceToHost, c_.stream));
    QTT_CUDA(cudaMemcpyAsync(pin + 1, c_.flags + 8, 4, cudaMemcpyDeviceToHost, c_.stream));
    c_.sync();
    unsigned long long ns;
    std::memcpy(&ns, pin, 8);
    int it;
    std::memcpy(&it, pin + 1, 4);
    iters = it;
    if (dbg) {
      unsigned long long ph[6];
      QTT_CUDA(cudaMemcpyAsync(ph, c_.scal + 32, sizeof(ph), cudaMemcpyDeviceToHost, c_.stream));
      c_.sync();
      std::fprintf(stderr, "[qtt] cg_fused dims %d,%d,%d R %d S3 %d tiles %d,%d composed %d grid %d iters %d: ns "
                   "step1 %llu step2 %llu step3 %llu red %llu upd %llu pupd %llu\n", L.lb, L.m, L.rb, L.R1, pl.S3,
                   100 * pl.p1_rb + pl.p1_cb, 100 * pl.p2_rb + pl.p2_cb, 1, grid, it, ph[0], ph[1], ph[2], ph[3],
                   ph[4], ph[5]);
    }
    const int calls = it + (xany ? 1 : 0);
    c_.stats.cg_iters += it;
    c_.stats.k1_calls += calls;
    c_.stats.k1_flops += kflops * calls;
    if (c_.profiling) {
      c_.stats.k1_ms += ns * 1e-6;
      c_.stats.k1_timed_flops += kflops * calls;
    }
    return u;
  }
  if (prm_.fused_cg) {
    // one persistent cooperative kernel for the whole CG solve (cg_fused.cu)
    const int grid = cg_fused_grid(c_.device);
    int S3 = 1, ktp = 1, tileA = 0, tile3 = 0;
    cg_fused_plan(L.lb, L.m, L.rb, L.R1, L.rk, grid, S3, ktp, tileA, tile3);
    // compose steps 1+2 into one GEMM phase when that costs at most ~15% more flops
    // (it saves a grid barrier and a pipeline fill per matvec); QTT_CG_COMPOSE=0/1 forces
    static const int compose_env = std::getenv("QTT_CG_COMPOSE") ? std::atoi(std::getenv("QTT_CG_COMPOSE")) : -1;
    const double f3 = cg_fused_flops(L.lb, L.lo, L.lk, L.m, L.n, L.R1, L.rb, L.rk, false);
    const double fc = cg_fused_flops(L.lb, L.lo, L.lk, L.m, L.n, L.R1, L.rb, L.rk, true);
    const bool composed = compose_env >= 0 ? compose_env != 0 : fc <= 1.15 * f3;
    DBuf t1(composed ? 1 : (long long)L.lb * L.lo * L.n * L.rk, c_.stream),
        t2((long long)L.lb * L.m * L.R1 * L.rk, c_.stream);
    DBuf bop(composed ? (long long)L.lb * L.m * L.R1 * L.lk * L.n : 1, c_.stream);
    if (composed) cg_fused_build_bop(L.phil, L.lb, L.lo, L.lk, L.Ap, L.m, L.n, L.R1, bop.p, c_.stream);
    DBuf part3((long long)S3 * dim, c_.stream), red(4LL * grid, c_.stream);
    CGFusedArgs a{};
    a.phil = L.phil; a.lb = L.lb; a.lo = L.lo; a.lk = L.lk;
    a.Ap = L.Ap; a.m = L.m; a.n = L.n; a.R1 = L.R1;
    a.phir = L.phir; a.rb = L.rb; a.rk = L.rk;
    a.b = rhs_p; a.invd = invd.p; a.x = u.p; a.r = r.p; a.z = z.p; a.p = p.p; a.q = q.p;
    a.Bop = composed ? bop.p : nullptr;
    a.t1 = t1.p; a.t2 = t2.p; a.part3 = part3.p; a.S3 = S3; a.kt_per3 = ktp; a.tileA = tileA; a.tile3 = tile3; a.red = red.p;
    a.dim = dim; a.atol = atol; a.maxiter = prm_.local_iter_cap; a.xany = xany ? 1 : 0;
    a.out_iters = c_.flags + 8;
    a.out_rnorm = c_.scal + 20;
    a.out_mv_ns = (unsigned long long*)(c_.scal + 21);
    QTT_CUDA(cudaMemsetAsync(c_.scal + 21, 0, 8, c_.stream));
    static const bool dbg = std::getenv("QTT_DEBUG") != nullptr;
    a.phase_ns = dbg ? (unsigned long long*)(c_.scal + 32) : nullptr;
    if (dbg) QTT_CUDA(cudaMemsetAsync(c_.scal + 32, 0, 6 * 8, c_.stream));
    cg_fused_launch(a, grid, c_.stream);
    double* pin = c_.host_scalars(2);
    QTT_CUDA(cudaMemcpyAsync(pin, c_.scal + 21, 8, cudaMemcpyDeviceToHost, c_.stream));
    QTT_CUDA(cudaMemcpyAsync(pin + 1, c_.flags + 8, 4, cudaMemcpyDeviceToHost, c_.stream));
    c_.sync();
    unsigned long long ns;
    std::memcpy(&ns, pin, 8);
    int it;
    std::memcpy(&it, pin + 1, 4);
    iters = it;
    if (dbg) {
      unsigned long long ph[6];
      QTT_CUDA(cudaMemcpyAsync(ph, c_.scal + 32, sizeof(ph), cudaMemcpyDeviceToHost, c_.stream));
      c_.sync();
      std::fprintf(stderr, "[qtt] cg_fused dims %d,%d,%d R %d S3 %d tiles %d,%d composed %d grid %d iters %d: ns "
                   "step1 %llu step2 %llu step3 %llu red %llu upd %llu pupd %llu\n", L.lb, L.m, L.rb, L.R1, S3,
                   tileA, tile3, composed ? 1 : 0, grid, it, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5]);
    }
    const int calls = it + (xany ? 1 : 0);
    c_.stats.cg_iters += it;
    c_.stats.k1_calls += calls;
    c_.stats.k1_flops += kflops * calls;
    if (c_.profiling) {
      c_.stats.k1_ms += ns * 1e-6;
      c_.stats.k1_timed_flops += kflops * calls;
    }
    return u;
  }
  int* flags = c_.flags;
  if (xany) {  // r = b - A x0
    const int t = c_.prof_begin();
    matvec(u.p, r.p, -1.0, 1.0, nullptr);
    c_.prof_end(t, 0, kflops);
    c_.stats.k1_calls++;
    c_.stats.k1_flops += kflops;
  }
  const int rb = (int)std::min<long long>(RB, cdiv(dim, 256));
  cg_start_kernel<<<rb, 256, 0, c_.stream>>>(r.p, invd.p, z.p, p.p, dim, atol, c_.red_partial,
                                             c_.red_counter, c_.scal, flags);
  QTT_CHECK_LAUNCH();
  const int maxiter = prm_.local_iter_cap;
  constexpr int CHUNK = 8;
  std::vector<int> tidx;
  int done_iters = 0;
  if (maxiter <= 0) {
    done_iters = 0;
  } else {
    for (int launched = 0; launched < maxiter;) {
      const int nlaunch = std::min(CHUNK, maxiter - launched);
      for (int i = 0; i < nlaunch; ++i) {
        const int t = c_.prof_begin();
        matvec(p.p, q.p, 1.0, 0.0, flags);
        c_.prof_end(t, 0, kflops);
        tidx.push_back(t);
        cg_alpha_kernel<<<rb, 256, 0, c_.stream>>>(p.p, q.p, dim, c_.red_partial, c_.red_counter, c_.scal,
                                                   flags);
        QTT_CHECK_LAUNCH();
        cg_update_kernel<<<rb, 256, 0, c_.stream>>>(u.p, r.p, z.p, p.p, q.p, invd.p, dim, atol, maxiter,
                                                    c_.red_partial, c_.red_counter, c_.scal, flags);
        QTT_CHECK_LAUNCH();
        cg_dir_kernel<<<grid_for(dim), 256, 0, c_.stream>>>(p.p, z.p, dim, c_.scal, flags);
        QTT_CHECK_LAUNCH();
      }
      launched += nlaunch;
      int* pin = (int*)c_.host_scalars(1);
      QTT_CUDA(cudaMemcpyAsync(pin, flags, 8, cudaMemcpyDeviceToHost, c_.stream));
      c_.sync();
      done_iters = pin[1];
      if (pin[0]) break;
    }
  }
  c_.stats.cg_iters += done_iters;
  c_.stats.k1_calls += done_iters;
  c_.stats.k1_flops += kflops * done_iters;
  iters = done_iters;
  // launches after convergence were no-ops (device skip flag): not K1 work
  for (int i = done_iters; i < (int)tidx.size(); ++i) c_.prof_discard(tidx[i]);
  (void)profile;
  return u;
}

namespace {

class Solver {
 public:
  Solver(Ctx& c, Train& A, const Train& f, const AmenParams& prm, DrawStream& draws)
      : c_(c), A_(A), f_(f), prm_(prm), draws_(draws) {
    K_ = A.order();
    dims_ = f.dims();
  }

  Train run(const Train* x0, AmenResult& res);
  // One core step on injected state (qtt_amen_step, the state-injected parity check).
  void step_injected(int sweep, int k, bool forward, double lam_max, double nf, const std::vector<HostArray>& in,
                     std::vector<HostArray>& out, StepInfo& info);

 private:
  Ctx& c_;
  Train& A_;
  const Train& f_;
  AmenParams prm_;
  DrawStream& draws_;
  int K_ = 0;
  std::vector<int> dims_;
  std::vector<Core> x_, z_;
  std::vector<Env> phi_, phiz_, psi_, psiz_;
  double lam_max_ = 0.0, nf_ = 0.0;
  int sweep_ = 0;
  double last_lam_ = 0.0;
  int last_rank_ = 0, last_iters_ = 0;

  void probe_symmetry();
  Train default_x0();
  std::vector<Core> init_z();
  void full_prepass(bool forward, bool xenvs, bool zenvs);
  double sweep(bool forward);
  bool core_step(bool forward, int k, double& est);
  void gather_state(int k, bool forward, bool after, std::vector<HostArray>& v);
  void maybe_dump(int k, bool forward, bool after);
  std::vector<HostArray> dump_in_;
  double dump_lam_in_ = 0.0;
  void env_step_left(int k, bool xenvs, bool zenvs);
  void env_step_right(int k, bool xenvs, bool zenvs);
  Env phi_left(const Env& phi, const Core& bra, int k, const Core& ket);
  Env phi_right(const Env& phi, const Core& bra, int k, const Core& ket);
  Env psi_left_(const Env& psi, const Core& bra, int k);
  Env psi_right_(const Env& psi, const Core& bra, int k);
  DBuf local_rhs_(const Env& pl, int k, const Env& pr);
  DBuf mixed_res(const Env& psl, int k, const Env& psr, const Env& pl, const DBuf& u, int rl, int rr,
                 const Env& pr);
  void matvec(const Env& pl, int k, const Env& pr, const double* v, double* y, double alpha,
              double beta, const int* skip, bool timed);
  DBuf solve_local(int k, const DBuf& rhs, const Core& prev, double& lam);
};

Env Solver::phi_left(const Env& phi, const Core& bra, int k, const Core& ket) {
  const Core& a = A_.cores[k];
  Env out;
  out.b = bra.r1; out.o = a.r1; out.k = ket.r1;
  out.d.alloc((long long)out.b * out.o * out.k, c_.stream);
  DBuf sc(env_left_scratch(phi.b, phi.o, phi.k, a.m, a.n, a.r1, ket.r1, bra.r1) +
              (long long)out.b * out.o * out.k * 4, c_.stream);
  const double fl = env_flops(phi.b, phi.o, phi.k, a.m, a.n, a.r1, bra.r1, ket.r1);
  const int t = c_.prof_begin();
  env_left(phi.d.p, phi.b, phi.o, phi.k, bra.d.p, bra.r1, A_.Ap[k].p, a.m, a.n, a.r1, ket.d.p, ket.r1,
           out.d.p, {sc.p, sc.n}, c_.stream);
  c_.prof_end(t, 1, fl);
  c_.stats.env_calls++;
  c_.stats.env_flops += fl;
  return out;
}

Env Solver::phi_right(const Env& phi, const Core& bra, int k, const Core& ket) {
  const Core& a = A_.cores[k];
  Env out;
  out.b = bra.r0; out.o = a.r0; out.k = ket.r0;
  out.d.alloc((long long)out.b * out.o * out.k, c_.stream);
  DBuf sc(env_right_scratch(phi.b, phi.o, phi.k, a.m, a.n, a.r0, ket.r0, bra.r0) +
              (long long)out.b * out.o * out.k * 4, c_.stream);
  const double fl = env_flops(phi.b, phi.o, phi.k, a.m, a.n, a.r0, bra.r0, ket.r0);
  const int t = c_.prof_begin();
  env_right(phi.d.p, phi.b, phi.o, phi.k, bra.d.p, bra.r0, A_.Aq[k].p, a.m, a.n, a.r0, ket.d.p, ket.r0,
            out.d.p, {sc.p, sc.n}, c_.stream);
  c_.prof_end(t, 1, fl);
  c_.stats.env_calls++;
  c_.stats.env_flops += fl;
  return out;
}

Env Solver::psi_left_(const Env& psi, const Core& bra, int k) {
  const Core& fk = f_.cores[k];
  Env out;
  out.b = bra.r1; out.o = fk.r1;
  out.d.alloc((long long)out.b * out.o, c_.stream);
  DBuf sc((long long)psi.b * fk.m * fk.r1 + (long long)out.b * out.o * 8, c_.stream);
  psi_left(psi.d.p, psi.b, psi.o, bra.d.p, bra.m, bra.r1, fk.d.p, fk.r1, out.d.p, {sc.p, sc.n}, c_.stream);
  return out;
}

Env Solver::psi_right_(const Env& psi, const Core& bra, int k) {
  const Core& fk = f_.cores[k];
  Env out;
  out.b = bra.r0; out.o = fk.r0;
  out.d.alloc((long long)out.b * out.o, c_.stream);
  DBuf sc((long long)fk.r0 * fk.m * psi.b + (long long)out.b * out.o * 8, c_.stream);
  psi_right(psi.d.p, psi.b, psi.o, bra.d.p, bra.r0, bra.m, fk.d.p, fk.r0, out.d.p, {sc.p, sc.n}, c_.stream);
  return out;
}

DBuf Solver::local_rhs_(const Env& pl, int k, const Env& pr) {
  const Core& fk = f_.cores[k];
  DBuf out((long long)pl.b * fk.m * pr.b, c_.stream);
  DBuf sc((long long)pl.b * fk.m * fk.r1 + (long long)pl.b * fk.m * pr.b * 8, c_.stream);
  local_rhs(pl.d.p, pl.b, pl.o, fk.d.p, fk.m, fk.r1, pr.d.p, pr.b, out.p, {sc.p, sc.n}, c_.stream);
  return out;
}

void Solver::matvec(const Env& pl, int k, const Env& pr, const double* v, double* y, double alpha,
                    double beta, const int* skip, bool timed) {
  const Core& a = A_.cores[k];
  const long long need = local_matvec_scratch(pl.b, pl.o, pl.k, a.m, a.n, a.r1, pr.b, pr.k) +
                         (long long)pl.b * a.m * pr.b * 8;
  DBuf sc(need, c_.stream);
  local_matvec(pl.d.p, pl.b, pl.o, pl.k, A_.Ap[k].p, a.m, a.n, a.r1, pr.d.p, pr.b, pr.k, v, y, alpha,
               beta, {sc.p, sc.n}, c_.stream, skip);
  (void)timed;
}

DBuf Solver::mixed_res(const Env& psl, int k, const Env& psr, const Env& pl, const DBuf& u, int rl,
                       int rr, const Env& pr) {
  (void)rl; (void)rr;
  DBuf out = local_rhs_(psl, k, psr);
  const Core& a = A_.cores[k];
  const double fl = local_matvec_flops(pl.b, pl.o, pl.k, a.m, a.n, a.r1, pr.b, pr.k);
  const int t = c_.prof_begin();
  matvec(pl, k, pr, u.p, out.p, -1.0, 1.0, nullptr, false);
  c_.prof_end(t, 0, fl);
  c_.stats.k1_calls++;
  c_.stats.k1_flops += fl;
  return out;
}

DBuf Solver::solve_local(int k, const DBuf& rhs, const Core& prev, double& lam) {
  const Env& pl = phi_[k];
  const Env& pr = phi_[k + 1];
  const Core& a = A_.cores[k];
  LocalSystem L{pl.d.p, pl.b, pl.o, pl.k, a.d.p, A_.Ap[k].p, a.r0, a.m, a.n, a.r1, pr.d.p, pr.b, pr.o, pr.k};
  int iters = 0;
  DBuf u = solve_local_system(c_, L, rhs.p, prev.d.p, prm_, sweep_, k, lam, iters, c_.profiling);
  last_iters_ = iters;
  const long long dim = (long long)pl.b * a.m * pr.b;
  const int path = (!prm_.local_iterative && dim <= prm_.direct_dim_cap) ? 0 : 1;
  c_.trace.push_back({sweep_, k, pl.b, a.m, pr.b, phiz_[k].b, phiz_[k + 1].b, a.r0, a.r1, path, iters});
  return u;
}

// ------------------------------------------------------------------ env plumbing
void Solver::env_step_left(int k, bool xenvs, bool zenvs) {
  if (xenvs) {
    phi_[k + 1] = phi_left(phi_[k], x_[k], k, x_[k]);
    psi_[k + 1] = psi_left_(psi_[k], x_[k], k);
  }
  if (zenvs) {
    phiz_[k + 1] = phi_left(phiz_[k], z_[k], k, x_[k]);
    psiz_[k + 1] = psi_left_(psiz_[k], z_[k], k);
  }
}

void Solver::env_step_right(int k, bool xenvs, bool zenvs) {
  if (xenvs) {
    phi_[k] = phi_right(phi_[k + 1], x_[k], k, x_[k]);
    psi_[k] = psi_right_(psi_[k + 1], x_[k], k);
  }
  if (zenvs) {
    phiz_[k] = phi_right(phiz_[k + 1], z_[k], k, x_[k]);
    psiz_[k] = psi_right_(psiz_[k + 1], z_[k], k);
  }
}

// amen.py:300-321.  The reference rebuilds every opposite-side environment at the
// start of each sweep; those equal the ones the previous sweep already produced
// (each depends only on cores that sweep no longer touches), so they are kept
// resident and only rebuilt when their inputs changed (first sweep, z redraw).
void Solver::full_prepass(bool forward, bool xenvs, bool zenvs) {
  if (forward)
    for (int k = K_ - 1; k >= 1; --k) env_step_right(k, xenvs, zenvs);
  else
    for (int k = 0; k < K_ - 1; ++k) env_step_left(k, xenvs, zenvs);
}

double Solver::sweep(bool forward) {
  double est = 0.0;
  for (int step = 0; step < K_; ++step) {
    const int k = forward ? step : K_ - 1 - step;
    maybe_dump(k, forward, false);
    const bool last = core_step(forward, k, est);
    maybe_dump(k, forward, true);
    if (last) break;
  }
  return est;
}

// Host copies of the step state: in = x_k, x_nb, z_k, phi_k, phi_k1, phiz_k, phiz_k1, psi_k,
// psi_k1, psiz_k, psiz_k1, A_k, f_k; after = x_k, x_nb, z_k and the four environments the step rebuilt
// (bond k+1 forward, bond k backward).  nb = k+1 forward, k-1 backward.
void Solver::gather_state(int k, bool forward, bool after, std::vector<HostArray>& v) {
  auto core = [&](const Core& c) {
    HostArray h;
    h.d0 = c.r0; h.d1 = c.m * c.n; h.d2 = c.r1;
    h.v.resize(c.numel());
    c.d.download(h.v.data(), c.numel());
    v.push_back(std::move(h));
  };
  auto env = [&](const Env& e) {
    HostArray h;
    h.d0 = e.b; h.d1 = e.o; h.d2 = e.k;
    h.v.resize((size_t)e.b * e.o * e.k);
    e.d.download(h.v.data(), (long long)h.v.size());
    v.push_back(std::move(h));
  };
  const int nb = forward ? k + 1 : k - 1;
  core(x_[k]);
  core(x_[nb]);
  core(z_[k]);
  if (!after) {
    for (auto* e : {&phi_, &phiz_}) { env((*e)[k]); env((*e)[k + 1]); }
    for (auto* e : {&psi_, &psiz_}) { env((*e)[k]); env((*e)[k + 1]); }
    core(A_.cores[k]);  // the operator and rhs cores of the step, as (r0, m*n, r1): the dump
    core(f_.cores[k]);  // is then self-contained (host assemblies can differ at round-off level)
  } else {
    const int b = forward ? k + 1 : k;
    env(phi_[b]); env(phiz_[b]); env(psi_[b]); env(psiz_[b]);
  }
  c_.sync();
}

// QTT_DUMP_STEP="sweep,core,path": write the state before and after that core step of the
// solve (QSTEP1 file, read by tests/golden_io.py) -- the input of the state-injected check.
void Solver::maybe_dump(int k, bool forward, bool after) {
  static const char* spec = std::getenv("QTT_DUMP_STEP");
  if (!spec) return;
  int ds = -1, dk = -1;
  char path[512] = {0};
  if (std::sscanf(spec, "%d,%d,%511s", &ds, &dk, path) != 3 || ds != sweep_ || dk != k) return;
  const bool lastk = forward ? (k == K_ - 1) : (k == 0);
  if (lastk) return;
  if (!after) {
    dump_in_.clear();
    gather_state(k, forward, false, dump_in_);
    dump_lam_in_ = lam_max_;
    return;
  }
  std::vector<HostArray> out;
  gather_state(k, forward, true, out);
  FILE* fh = std::fopen(path, "wb");
  if (!fh) throw Error(QTT_ERR_ARG, std::string("cannot write ") + path);
  const int hdr[7] = {sweep_, k, forward ? 1 : 0, last_rank_, last_iters_, (int)dump_in_.size(), (int)out.size()};
  const double sc[3] = {dump_lam_in_, nf_, last_lam_};
  std::fwrite("QSTEP1", 1, 6, fh);
  std::fwrite(hdr, sizeof(int), 7, fh);
  std::fwrite(sc, sizeof(double), 3, fh);
  for (auto* vv : {&dump_in_, &out})
    for (auto& h : *vv) {
      const int d[3] = {h.d0, h.d1, h.d2};
      std::fwrite(d, sizeof(int), 3, fh);
      std::fwrite(h.v.data(), sizeof(double), h.v.size(), fh);
    }
  std::fclose(fh);
  std::fprintf(stderr, "[qtt] dumped core step (sweep %d, core %d) to %s\n", sweep_, k, path);
}

void Solver::step_injected(int sweep, int k, bool forward, double lam_max, double nf, const std::vector<HostArray>& in,
                           std::vector<HostArray>& out, StepInfo& info) {
  if (k < 0 || k >= K_) throw Error(QTT_ERR_ARG, "step core out of range");
  if (forward ? (k == K_ - 1) : (k == 0)) throw Error(QTT_ERR_ARG, "state-injected step needs a neighbour core");
  if (in.size() < 11) throw Error(QTT_ERR_ARG, "state-injected step takes 11 state arrays");
  prepare_operator(c_, A_);
  x_.resize(K_);
  z_.resize(K_);
  for (auto* e : {&phi_, &phiz_, &psi_, &psiz_}) e->resize(K_ + 1);
  auto core = [&](const HostArray& h) {
    Core c = make_core(c_, h.d0, h.d1, 1, h.d2);
    c.d.upload(h.v.data(), c.numel());
    return c;
  };
  auto env = [&](const HostArray& h) {
    Env e;
    e.b = h.d0; e.o = h.d1; e.k = h.d2;
    e.d.alloc((long long)h.v.size(), c_.stream);
    e.d.upload(h.v.data(), (long long)h.v.size());
    return e;
  };
  const int nb = forward ? k + 1 : k - 1;
  x_[k] = core(in[0]);
  x_[nb] = core(in[1]);
  z_[k] = core(in[2]);
  phi_[k] = env(in[3]); phi_[k + 1] = env(in[4]);
  phiz_[k] = env(in[5]); phiz_[k + 1] = env(in[6]);
  psi_[k] = env(in[7]); psi_[k + 1] = env(in[8]);
  psiz_[k] = env(in[9]); psiz_[k + 1] = env(in[10]);
  const Core& a = A_.cores[k];
  if (x_[k].m != a.n || phi_[k].o != a.r0 || phi_[k + 1].o != a.r1 || phi_[k].k != x_[k].r0 ||
      phi_[k + 1].k != x_[k].r1 || psi_[k].o != f_.cores[k].r0 || psi_[k + 1].o != f_.cores[k].r1)
    throw Error(QTT_ERR_SHAPE, "state-injected step: state does not fit the operator/rhs cores");
  sweep_ = sweep;
  lam_max_ = lam_max;
  nf_ = nf;
  double est = 0.0;
  info.last = core_step(forward, k, est);
  info.lam = last_lam_;
  info.rank = last_rank_;
  info.iters = last_iters_;
  info.est = est;
  out.clear();
  gather_state(k, forward, true, out);
}

// The per-core body of _sweep (amen.py:324-390); returns true at the last core of the pass.
bool Solver::core_step(bool forward, int k, double& est) {
  const double rel = prm_.round_tol;
  const int cap = prm_.round_max_rank;
  {
    const int rl = x_[k].r0, m = x_[k].m, rr = x_[k].r1;
    DBuf rhs = local_rhs_(psi_[k], k, psi_[k + 1]);
    double lam = 0.0;
    c_.phase((!prm_.local_iterative && (long long)rl * m * rr <= prm_.direct_dim_cap) ? PH_DIRECT : PH_CG);
    DBuf u = solve_local(k, rhs, x_[k], lam);
    c_.phase(PH_MIXED);
    last_lam_ = lam;
    lam_max_ = std::max(lam_max_, lam);
    const bool have_dabs = K_ > 1 && lam_max_ > 0;
    const double dabs = have_dabs ? prm_.residual_tol * nf_ / (lam_max_ * std::sqrt((double)(K_ - 1))) : 0.0;

    // zeta: local residual in the z bases (rz_l, m, rz_r)
    DBuf zeta = mixed_res(psiz_[k], k, psiz_[k + 1], phiz_[k], u, rl, rr, phiz_[k + 1]);
    const int zl = phiz_[k].b, zr = phiz_[k + 1].b;
    const bool last = forward ? (k == K_ - 1) : (k == 0);
    if (last) {
      Core nu;
      nu.r0 = rl; nu.m = m; nu.n = 1; nu.r1 = rr;
      nu.d = std::move(u);
      x_[k] = std::move(nu);
      Core nz;
      nz.r0 = zl; nz.m = m; nz.n = 1; nz.r1 = zr;
      nz.d = std::move(zeta);
      nrm2(c_, nz.d.p, nz.numel(), c_.scal + 12);
      z_[k] = std::move(nz);
      read_scalars(c_, c_.scal + 12, 1, &est);
      last_rank_ = rr;
      return true;
    }

    // enrichment from the mixed x/z residual, and the truncated split of u
    DBuf enr;
    int rows, cols, ecols;
    CMatView uview, eview;
    if (forward) {
      enr = mixed_res(psi_[k], k, psiz_[k + 1], phi_[k], u, rl, rr, phiz_[k + 1]);  // (rl, m, zr)
      rows = rl * m; cols = rr; ecols = zr;
      uview = crowmajor(u.p, rows, cols);
      eview = crowmajor(enr.p, rows, ecols);
    } else {
      enr = mixed_res(psiz_[k], k, psi_[k + 1], phiz_[k], u, rl, rr, phi_[k + 1]);  // (zl, m, rr)
      rows = m * rr; cols = rl; ecols = zl;
      uview = ctrans(crowmajor(u.p, rl, m * rr));
      eview = ctrans(crowmajor(enr.p, zl, m * rr));
    }
    const int kk = std::min(rows, cols);
    DBuf U((long long)rows * kk, c_.stream), s(kk, c_.stream), Vt((long long)kk * cols, c_.stream);
    c_.phase(PH_SVD);
    svd(c_, uview, rowmajor(U.p, rows, kk), s.p, rowmajor(Vt.p, kk, cols));
    std::vector<double> hs(kk);
    read_scalars(c_, s.p, kk, hs.data());
    double norm = 0.0;
    for (double v : hs) norm += v * v;
    norm = std::sqrt(norm);
    int r;
    DBuf w;
    if (norm == 0.0) {  // amen.py:225-226
      r = 1;
      w.alloc(cols, c_.stream);
      fill(c_, w.p, cols, 0.0);
    } else {
      double delta = rel * norm;
      if (have_dabs) delta = std::min(delta, dabs);
      r = rank_for_tolerance(hs.data(), kk, delta);
      if (cap > 0) r = std::min(r, cap);
      r = std::max(r, 1);
      w.alloc((long long)r * cols, c_.stream);
      scale_rows(c_, Vt.p, cols, s.p, r, cols, w.p, cols);
    }
    last_rank_ = r;
    // q, R = qr([Q | enrich])
    const int acols = r + ecols;
    DBuf aug((long long)rows * acols, c_.stream);
    build_aug_kernel<<<grid_for((long long)rows * acols), 256, 0, c_.stream>>>(U.p, kk, r, eview, aug.p, rows);
    QTT_CHECK_LAUNCH();
    const int kq = std::min(rows, acols);
    DBuf Q((long long)rows * kq, c_.stream), R((long long)kq * acols, c_.stream);
    c_.phase(PH_QR);
    qr(c_, crowmajor(aug.p, rows, acols), rowmajor(Q.p, rows, kq), rowmajor(R.p, kq, acols));
    // absorb = R[:, :r] @ w   (kq x cols)
    DBuf absorb((long long)kq * cols, c_.stream);
    {
      GemmArgs g;
      g.M = kq; g.N = cols; g.K = r;
      gemm_set_A(g, R.p, acols, false);
      gemm_set_B(g, w.p, cols, false);
      gemm_set_C(g, absorb.p, cols);
      gemm(g, c_.stream);
    }
    // z core from qr(zeta)
    if (forward) {
      const int zrows = zl * m, kz = std::min(zrows, zr);
      Core nz = make_core(c_, zl, m, 1, kz);
      qr(c_, crowmajor(zeta.p, zrows, zr), rowmajor(nz.d.p, zrows, kz), MatView{});
      z_[k] = std::move(nz);
      // x_k = q (rl, m, kq);  x_{k+1} = absorb @ x_{k+1}
      Core nx;
      nx.r0 = rl; nx.m = m; nx.n = 1; nx.r1 = kq;
      nx.d = std::move(Q);
      x_[k] = std::move(nx);
      Core& nxt = x_[k + 1];
      Core nn = make_core(c_, kq, nxt.m, 1, nxt.r1);
      GemmArgs g;
      g.M = kq; g.N = nxt.m * nxt.r1; g.K = cols;
      gemm_set_A(g, absorb.p, cols, false);
      gemm_set_B(g, nxt.d.p, (long long)nxt.m * nxt.r1, false);
      gemm_set_C(g, nn.d.p, (long long)nxt.m * nxt.r1);
      gemm(g, c_.stream);
      x_[k + 1] = std::move(nn);
      c_.phase(PH_ENV);
      env_step_left(k, true, true);
      c_.phase(PH_RHS);
    } else {
      const int zcols = m * zr, kz = std::min(zcols, zl);
      Core nz = make_core(c_, kz, m, 1, zr);
      // qr(zeta.reshape(zl, m zr).T); z core = Q^T written directly
      qr(c_, ctrans(crowmajor(zeta.p, zl, zcols)), MatView{nz.d.p, zcols, kz, 1, zcols}, MatView{});
      z_[k] = std::move(nz);
      // x_k = q^T (kq, m, rr)
      Core nx = make_core(c_, kq, m, 1, rr);
      copy_view(c_, ctrans(crowmajor(Q.p, rows, kq)), rowmajor(nx.d.p, kq, rows));
      x_[k] = std::move(nx);
      // x_{k-1} = x_{k-1} @ absorb^T   ((r0' m') x rl) @ (rl x kq)
      Core& prv = x_[k - 1];
      Core np = make_core(c_, prv.r0, prv.m, 1, kq);
      GemmArgs g;
      g.M = prv.r0 * prv.m; g.N = kq; g.K = cols;
      gemm_set_A(g, prv.d.p, cols, false);
      gemm_set_B(g, absorb.p, cols, true);
      gemm_set_C(g, np.d.p, kq);
      gemm(g, c_.stream);
      x_[k - 1] = std::move(np);
      c_.phase(PH_ENV);
      env_step_right(k, true, true);
      c_.phase(PH_RHS);
    }
  }
  return false;
}

// ------------------------------------------------------------------ driver pieces
void Solver::probe_symmetry() {  // amen.py:249-272
  const std::vector<int> cd = A_.dims();
  auto random_vec = [&]() {
    Train v;
    for (int k = 0; k < K_; ++k) {
      const int r0 = k == 0 ? 1 : 2, r1 = k == K_ - 1 ? 1 : 2;
      Core core = make_core(c_, r0, cd[k], 1, r1);
      const double* h = draws_.take(core.numel());
      core.d.upload(h, core.numel());
      v.cores.push_back(std::move(core));
    }
    const double nv = tt_norm(c_, v);
    if (nv > 0) {
      Train s = tt_scale_copy(c_, v, 1.0 / nv);
      return s;
    }
    return v;
  };
  for (int it = 0; it < 2; ++it) {
    Train u = random_vec();
    Train v = random_vec();
    Train au = tt_apply(c_, A_, u);
    Train av = tt_apply(c_, A_, v);
    const double s1 = tt_dot(c_, v, au), s2 = tt_dot(c_, u, av);
    const double scale = tt_norm(c_, au) + tt_norm(c_, av) + 1e-300;
    if (std::fabs(s1 - s2) > 1e-6 * scale)
      throw Error(QTT_ERR_SOLVER,
                  "operator is not symmetric (<v,Au> != <u,Av> on random probes); assemble the "
                  "system with the symmetric boundary projection P A P + (I - P) before solving");
  }
}

Train Solver::default_x0() {  // amen.py:237-246
  Train diag;
  for (auto& a : A_.cores) {
    Core d = make_core(c_, a.r0, a.m, 1, a.r1);
    op_core_diag(c_, a.d.p, a.r0, a.m, a.r1, d.d.p);
    diag.cores.push_back(std::move(d));
  }
  Train ones = tt_ones(c_, dims_);
  double n = 1.0;
  for (int d : dims_) n *= d;
  const double mean_diag = tt_dot(c_, diag, ones) / n;
  if (std::fabs(mean_diag) < 1e-300) return tt_round(c_, f_, 1e-12, 8);
  const double mean_f = tt_dot(c_, f_, ones) / n;
  return tt_ones(c_, dims_, mean_f / mean_diag);
}

std::vector<Core> Solver::init_z() {  // amen.py:275-284
  std::vector<int> rk(K_ + 1, prm_.enrichment_rank);
  rk[0] = rk[K_] = 1;
  for (int k = 1; k < K_; ++k) {
    // cap = min(prod(dims[:k]), prod(dims[k:])), computed without overflow
    double left = 1, right = 1;
    for (int j = 0; j < k; ++j) left *= dims_[j];
    for (int j = k; j < K_; ++j) right *= dims_[j];
    const double cap = std::min(left, right);
    if (cap < rk[k]) rk[k] = (int)cap;
  }
  Train t;
  for (int k = 0; k < K_; ++k) {
    Core core = make_core(c_, rk[k], dims_[k], 1, rk[k + 1]);
    const double* h = draws_.take(core.numel());
    core.d.upload(h, core.numel());
    t.cores.push_back(std::move(core));
  }
  orthogonalize_rl(c_, t);
  return std::move(t.cores);
}

Train Solver::run(const Train* x0, AmenResult& res) {
  nf_ = tt_norm(c_, f_);
  if (nf_ == 0.0) {
    res.converged = true;
    res.sweeps_used = 0;
    res.final_residual = 0.0;
    return tt_zero(c_, dims_);
  }
  prepare_operator(c_, A_);
  probe_symmetry();
  Train start = x0 ? clone(c_, *x0) : default_x0();
  orthogonalize_rl(c_, start);
  if (tt_norm(c_, start) == 0.0) {
    start = tt_ones(c_, dims_, nf_);
    orthogonalize_rl(c_, start);
  }
  x_ = std::move(start.cores);
  z_ = init_z();

  phi_.resize(K_ + 1);
  phiz_.resize(K_ + 1);
  psi_.resize(K_ + 1);
  psiz_.resize(K_ + 1);
  for (auto* v : {&phi_, &phiz_}) {
    (*v)[0] = unit_env(c_);
    (*v)[K_] = unit_env(c_);
  }
  for (auto* v : {&psi_, &psiz_}) {
    (*v)[0] = unit_env(c_);
    (*v)[K_] = unit_env(c_);
  }

  const double tol = prm_.residual_tol;
  lam_max_ = 0.0;
  bool converged = false, have_final = false;
  double final_res = 0.0, best = INFINITY;
  int strikes = 0, last_check = -10;
  bool x_envs_valid = false, z_envs_valid = false;
  for (int sw = 1; sw <= prm_.max_sweeps; ++sw) {
    sweep_ = sw;
    const bool forward = (sw % 2 == 1);
    c_.phase(PH_PREPASS);
    if (!x_envs_valid || !z_envs_valid) full_prepass(forward, !x_envs_valid, !z_envs_valid);
    c_.phase(PH_RHS);
    const double est = sweep(forward);
    x_envs_valid = z_envs_valid = true;
    c_.stats.sweeps++;
    c_.prof_flush();
    std::vector<int> rk{1};
    for (auto& cc : x_) rk.push_back(cc.r1);
    res.rank_history.push_back(rk);
    res.residual_history.push_back(est / nf_);
    const auto& rh = res.residual_history;
    const bool cert = est / nf_ <= tol;
    bool plateau = false;
    if (prm_.stagnation_strikes > 0 && rh.size() >= 8) {
      const double a = *std::min_element(rh.end() - 4, rh.end());
      const double b = *std::min_element(rh.end() - 8, rh.end() - 4);
      plateau = a > 0.97 * b;
    }
    const bool spaced = sw - last_check >= 5;
    if (!cert && !(plateau && spaced)) continue;
    Train xcur;
    xcur.cores.reserve(K_);
    for (auto& cc : x_) {  // non-owning view is not expressible with DBuf; copy is cheap (cores)
      Core cp = make_core(c_, cc.r0, cc.m, cc.n, cc.r1);
      QTT_CUDA(cudaMemcpyAsync(cp.d.p, cc.d.p, cc.numel() * 8, cudaMemcpyDeviceToDevice, c_.stream));
      xcur.cores.push_back(std::move(cp));
    }
    bool gram = false;
    c_.phase(PH_CERT);
    const auto tc0 = std::chrono::steady_clock::now();
    final_res = residual_norm(c_, A_, xcur, f_, &gram);
    if (std::getenv("QTT_DEBUG"))
      std::fprintf(stderr, "[qtt] sweep %d certification %.6g (%s) %.3f s, max rank %d\n", sw, final_res,
                   gram ? "gram" : "exact",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count(),
                   *std::max_element(rk.begin(), rk.end()));
    c_.phase(PH_OTHER);
    (gram ? res.certifications_gram : res.certifications_exact)++;
    have_final = true;
    if (final_res <= tol) {
      converged = true;
      break;
    }
    if (!cert && spaced) {
      if (final_res > 0.97 * best) {
        strikes++;
        if (strikes >= prm_.stagnation_strikes) break;
        z_ = init_z();  // fresh enrichment directions (amen.py:485)
        z_envs_valid = false;
      } else {
        strikes = 0;
      }
      last_check = sw;
    }
    best = std::min(best, final_res);
  }
  res.sweeps_used = (int)res.rank_history.size();
  c_.prof_flush();
  Train x;
  x.cores = std::move(x_);
  if (!have_final || !converged) {
    bool gram = false;
    final_res = residual_norm(c_, A_, x, f_, &gram);
    (gram ? res.certifications_gram : res.certifications_exact)++;
    converged = final_res <= tol;
  }
  res.converged = converged;
  res.final_residual = final_res;
  return x;
}

}  // namespace

Train amen_solve(Ctx& c, Train& A, const Train& f, const Train* x0, const AmenParams& prm,
                 DrawStream& draws, AmenResult& res) {
  Solver s(c, A, f, prm, draws);
  return s.run(x0, res);
}

void amen_core_step(Ctx& c, Train& A, const Train& f, const AmenParams& prm, int sweep, int k, bool forward,
                    double lam_max, double f_norm, const std::vector<HostArray>& in, std::vector<HostArray>& out,
                    StepInfo& info) {
  DrawStream none;
  Solver s(c, A, f, prm, none);
  s.step_injected(sweep, k, forward, lam_max, f_norm, in, out, info);
}

}  // namespace qtt
