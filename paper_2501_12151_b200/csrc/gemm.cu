// FP64 DMMA GEMM (see gemm.cuh for the operand convention).
#include "gemm.cuh"

#include <algorithm>

namespace qtt {
namespace {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
struct Cfg {
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int LDA = BM + 4;  // == 4 (mod 16) doubles: conflict-free fragment loads
  static constexpr int LDB = BN + 4;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MI = WTM / 8, NI = WTN / 8;
  static constexpr size_t SMEM = (size_t)STAGES * BK * (LDA + LDB) * sizeof(double);
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert((BM * BK) % NT == 0 && (BN * BK) % NT == 0, "tile loads must divide evenly");
  static_assert(BK % 4 == 0 && BM % 4 == 0 && BN % 4 == 0, "4x4 swizzle");
};

// Element index e of a (BK x BX) tile -> (kk, xx).  When the global operand is
// contiguous along X, consecutive threads walk X (coalesced, conflict-free STS).
// Otherwise (contiguous along K) a 4x4 micro-block swizzle keeps 32-byte global
// sectors and spreads the 16 lanes of a half-warp over 16 distinct banks.
template <int BK>
__device__ __forceinline__ void tile_coord(int e, bool x_contig, int BX, int& kk, int& xx) {
  if (x_contig) {
    xx = e % BX;
    kk = e / BX;
  } else {
    int kq = e & 3, xq = (e >> 2) & 3, blk = e >> 4;
    kk = (blk % (BK / 4)) * 4 + kq;
    xx = (blk / (BK / 4)) * 4 + xq;
  }
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32)
    dgemm_kernel(GemmArgs g, int splits, int kt_per_split, double* __restrict__ ws) {
  using C_ = Cfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES>;
  constexpr int NT = C_::NT, LDA = C_::LDA, LDB = C_::LDB, MI = C_::MI, NI = C_::NI;
  extern __shared__ double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * BK * LDA;

  if (g.skip != nullptr && *g.skip != 0) return;
  if (g.lower_only && (int)(blockIdx.x * BN) >= (int)(blockIdx.y * BM + BM)) return;
  int z = blockIdx.z;
  const int split = z % splits;
  z /= splits;
  const int b1 = z % g.batch1;
  const int b2 = z / g.batch1;
  const double* __restrict__ A = g.A + b1 * g.a_bs1 + b2 * g.a_bs2;
  const double* __restrict__ B = g.B + b1 * g.b_bs1 + b2 * g.b_bs2;
  const int M = g.M, N = g.N, K = g.K;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int ktiles = (K + BK - 1) / BK;
  const int kt_begin = split * kt_per_split;
  const int kt_end = min(ktiles, kt_begin + kt_per_split);
  const bool a_mc = (g.a_rs == 1);
  const bool b_nc = (g.b_cs == 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp % WARPS_M) * C_::WTM;
  const int wn0 = (warp / WARPS_M) * C_::WTN;
  const int lr = lane >> 2, lc = lane & 3;

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_tile = [&](int kt, int stage) {
    const int k0 = kt * BK;
    double* dA = sA + stage * BK * LDA;
    double* dB = sB + stage * BK * LDB;
#pragma unroll
    for (int i = 0; i < (BM * BK) / NT; ++i) {
      int kk, mm;
      tile_coord<BK>(threadIdx.x + i * NT, a_mc, BM, kk, mm);
      const int gm = m0 + mm, gk = k0 + kk;
      const bool ok = gm < M && gk < K;
      const double* src = ok ? A + (long long)gm * g.a_rs + (long long)gk * g.a_cs : A;
      cp_async8(dA + kk * LDA + mm, src, ok);
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / NT; ++i) {
      int kk, nn;
      tile_coord<BK>(threadIdx.x + i * NT, b_nc, BN, kk, nn);
      const int gn = n0 + nn, gk = k0 + kk;
      const bool ok = gn < N && gk < K;
      const double* src = ok ? B + (long long)gk * g.b_rs + (long long)gn * g.b_cs : B;
      cp_async8(dB + kk * LDB + nn, src, ok);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (kt_begin + s < kt_end) load_tile(kt_begin + s, s);
    cp_async_commit();
  }

  for (int kt = kt_begin; kt < kt_end; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int stage = (kt - kt_begin) % STAGES;
    const int nk = kt + STAGES - 1;
    if (nk < kt_end) load_tile(nk, (nk - kt_begin) % STAGES);
    cp_async_commit();

    const double* cA = sA + stage * BK * LDA;
    const double* cB = sB + stage * BK * LDB;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = cA[(ks + lc) * LDA + wm0 + i * 8 + lr];
#pragma unroll
      for (int j = 0; j < NI; ++j) bf[j] = cB[(ks + lc) * LDB + wn0 + j * 8 + lr];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  if (splits > 1) {
    double* W = ws + (long long)split * M * N;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int row = m0 + wm0 + i * 8 + lr;
        const int col = n0 + wn0 + j * 8 + lc * 2;
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (row < M && col + t < N) W[(long long)row * N + col + t] = acc[i][j][t];
      }
    return;
  }
  double* C = g.C + b1 * g.c_bs1 + b2 * g.c_bs2;
  const double alpha = g.alpha, beta = g.beta;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int row = m0 + wm0 + i * 8 + lr;
      const int col = n0 + wn0 + j * 8 + lc * 2;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (row < M && col + t < N && (!g.lower_only || col + t <= row)) {
          double* p = C + (long long)row * g.c_rs + (long long)(col + t) * g.c_cs;
          double v = alpha * acc[i][j][t];
          if (beta != 0.0) v = fma(beta, *p, v);
          *p = v;
        }
      }
    }
}

__global__ void splitk_reduce(const double* __restrict__ ws, int splits, int M, int N, double* C,
                              long long c_rs, long long c_cs, double alpha, double beta,
                              const int* skip) {
  if (skip != nullptr && *skip != 0) return;
  const long long total = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += ws[k * total + e];  // fixed order: deterministic
    const int row = (int)(e / N), col = (int)(e % N);
    double* p = C + row * c_rs + col * c_cs;
    double v = alpha * s;
    if (beta != 0.0) v = fma(beta, *p, v);
    *p = v;
  }
}

template <int BM, int BN, int BK, int WM, int WN, int ST>
void launch(const GemmArgs& g, int splits, int kt_per, double* ws, cudaStream_t s) {
  using C_ = Cfg<BM, BN, BK, WM, WN, ST>;
  static bool attr_set = false;  // per-instantiation, set once per process
  if (!attr_set) {
    QTT_CUDA(cudaFuncSetAttribute(dgemm_kernel<BM, BN, BK, WM, WN, ST>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C_::SMEM));
    attr_set = true;
  }
  long long zb = (long long)g.batch1 * g.batch2 * splits;
  if (zb > 65535) throw Error(QTT_ERR_ARG, "gemm: batch too large for grid.z");
  dim3 grid(cdiv(g.N, BN), cdiv(g.M, BM), (unsigned)zb);
  dgemm_kernel<BM, BN, BK, WM, WN, ST><<<grid, C_::NT, C_::SMEM, s>>>(g, splits, kt_per, ws);
  QTT_CHECK_LAUNCH();
}

constexpr int kSMs = 148;

struct Plan {
  int cfg;      // 0: 64x64, 1: 32x32, 2: 128x64
  int splits;
  int kt_per;
};

Plan plan_for(const GemmArgs& g) {
  Plan p{0, 1, 0};
  const long long batch = (long long)g.batch1 * g.batch2;
  if (g.M <= 40 || g.N <= 40)
    p.cfg = 1;
  else if (g.M >= 512 && (long long)cdiv(g.M, 128) * cdiv(g.N, 64) * batch >= 2 * kSMs)
    p.cfg = 2;
  const int bm = p.cfg == 1 ? 32 : (p.cfg == 2 ? 128 : 64);
  const int bn = p.cfg == 1 ? 32 : 64;
  const long long tiles = (long long)cdiv(g.M, bm) * cdiv(g.N, bn) * batch;
  const int ktiles = cdiv(g.K, 16);
  p.kt_per = ktiles;
  if (batch == 1 && tiles < kSMs && ktiles >= 16) {
    int want = (int)std::min<long long>(cdiv(2 * kSMs, tiles), ktiles / 8);
    if (want > 1) {
      p.kt_per = cdiv(ktiles, want);
      p.splits = cdiv(ktiles, p.kt_per);
    }
  }
  return p;
}

}  // namespace

long long gemm_workspace_hint(const GemmArgs& g) {
  Plan p = plan_for(g);
  return p.splits > 1 ? (long long)p.splits * g.M * g.N : 0;
}

void gemm(const GemmArgs& g, cudaStream_t s, double* ws, long long ws_doubles) {
  if (g.M <= 0 || g.N <= 0) return;
  if (g.K <= 0) {
    // C = beta*C (alpha * empty sum): reuse the reduce kernel with zero splits
    const long long total = (long long)g.M * g.N;
    for (int b2 = 0; b2 < g.batch2; ++b2)
      for (int b1 = 0; b1 < g.batch1; ++b1) {
        double* C = g.C + b1 * g.c_bs1 + b2 * g.c_bs2;
        splitk_reduce<<<cdiv(total, 256), 256, 0, s>>>(nullptr, 0, g.M, g.N, C, g.c_rs, g.c_cs, 0.0, g.beta, g.skip);
        QTT_CHECK_LAUNCH();
      }
    return;
  }
  Plan p = plan_for(g);
  if (g.lower_only) {
    p.splits = 1;
    p.kt_per = cdiv(g.K, 16);
  }
  if (p.splits > 1 && (ws == nullptr || ws_doubles < (long long)p.splits * g.M * g.N)) {
    p.splits = 1;
    p.kt_per = cdiv(g.K, 16);
  }
  switch (p.cfg) {
    case 1: launch<32, 32, 16, 2, 2, 4>(g, p.splits, p.kt_per, ws, s); break;
    case 2: launch<128, 64, 16, 4, 2, 3>(g, p.splits, p.kt_per, ws, s); break;
    default: launch<64, 64, 16, 2, 2, 3>(g, p.splits, p.kt_per, ws, s); break;
  }
  if (p.splits > 1) {
    const long long total = (long long)g.M * g.N;
    int blocks = (int)std::min<long long>(cdiv(total, 256), 4 * kSMs);
    splitk_reduce<<<blocks, 256, 0, s>>>(ws, p.splits, g.M, g.N, g.C, g.c_rs, g.c_cs, g.alpha, g.beta, g.skip);
    QTT_CHECK_LAUNCH();
  }
}

}  // namespace qtt
