// TMA-fed DMMA GEMM for K-contiguous operands (C = alpha A B^T + beta C with A [M][K] and
// B [N][K] row-major): persistent CTAs (2 per SM) stream output tiles of 128 x 64 through
// a 3-stage 128B-swizzled cp.async.bulk.tensor ring (tma_tile.cuh), DMMA + LDS only in the
// main loop.  Short-output / long-K products are split along K into one full wave of
// items whose partials are summed in a fixed order (deterministic).  Measured in
// isolation (tools/tile_bench.cu): 29.6-32.5 TF/s against 27 TF/s of the cp.async engine.
#include <algorithm>
#include <cmath>

#include "gemm.cuh"
#include "gemm_tma.cuh"
#include "tma_tile.cuh"

namespace qtt {
namespace {

using TC = tma::Cfg<128, 64, 4, 2, 3>;
constexpr int kSMs = 148;
constexpr int kPerSM = 2;

struct TmaGemmArgs {
  CUtensorMap ma, mb;
  int M, N, K;
  int tn;           // output tiles along N
  int tiles;        // output tiles
  int splits, kt_per;
  double* C;        // splits == 1: row-major, ldc
  long long ldc;
  double alpha, beta;
  double* ws;       // splits > 1: splits x M x N partials
};

__global__ void __launch_bounds__(TC::NT) tma_gemm_kernel(const __grid_constant__ TmaGemmArgs a) {
  extern __shared__ unsigned char smem_raw[];
  tma::Ring ring = tma::ring_init<TC::STAGES>(smem_raw);
  if (threadIdx.x == 0) {
    tma::prefetch_map(&a.ma);
    tma::prefetch_map(&a.mb);
  }
  const int items = a.tiles * a.splits;
  const int mine = items > (int)blockIdx.x ? (items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int KT = (a.K + 15) / 16;
  auto get = [&](int i) {
    const int it = blockIdx.x + i * gridDim.x;
    const int s = it % a.splits, t = it / a.splits;
    tma::Item r;
    r.ma = &a.ma;
    r.mb = &a.mb;
    r.m0 = (t / a.tn) * TC::BM;
    r.n0 = (t % a.tn) * TC::BN;
    r.kb = s * a.kt_per;
    r.ke = min(KT, r.kb + a.kt_per);
    return r;
  };
  auto epi = [&](const tma::Item& it, const double (&acc)[TC::MI][TC::NI][2]) {
    if (a.splits == 1) {
      tma::for_each<TC>(it.m0, it.n0, a.M, a.N, acc, [&](int r, int c, double v) {
        double* p = a.C + (long long)r * a.ldc + c;
        double o = a.alpha * v;
        if (a.beta != 0.0) o = fma(a.beta, *p, o);
        *p = o;
      });
    } else {
      double* W = a.ws + (long long)(it.kb / a.kt_per) * a.M * a.N;
      tma::for_each<TC>(it.m0, it.n0, a.M, a.N, acc,
                        [&](int r, int c, double v) { W[(long long)r * a.N + c] = v; });
    }
  };
  tma::stream<TC>(ring, mine, get, epi);
}

__global__ void tma_splitk_reduce(const double* __restrict__ ws, int splits, int M, int N, double* C, long long ldc,
                                  double alpha, double beta) {
  const long long total = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += ws[k * total + e];  // fixed order: deterministic
    double* p = C + (e / N) * ldc + (e % N);
    double v = alpha * s;
    if (beta != 0.0) v = fma(beta, *p, v);
    *p = v;
  }
}

}  // namespace

bool gemm_tma_eligible(const GemmArgs& g) {
  if (g.batch1 != 1 || g.batch2 != 1 || g.lower_only || g.skip != nullptr) return false;
  if (g.a_cs != 1 || g.b_rs != 1 || g.c_cs != 1) return false;  // A [M][K], B [N][K], C [M][N]
  if (g.K < 64 || g.M < 64 || g.N < 32) return false;
  if ((double)g.M * g.N * g.K < (double)(1 << 24)) return false;  // small products: cp.async engine
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(g.A) || !al(g.B) || (g.a_rs & 1) || (g.b_cs & 1)) return false;
  return true;
}

TmaGemmPlan gemm_tma_plan(const GemmArgs& g) {
  TmaGemmPlan p;
  const int tiles = cdiv(g.M, TC::BM) * cdiv(g.N, TC::BN);
  const int KT = cdiv(g.K, 16);
  const int slots = kSMs * kPerSM;
  double best = 1e300;
  for (int s = 1; s <= std::max(1, KT / 4); ++s) {
    const int kt = cdiv(KT, s);
    const int S = cdiv(KT, kt);
    if (S != s && s > 1) continue;
    const double waves = std::ceil((double)tiles * S / slots);
    // per item: ~2 k-tiles of ramp; partials: write + read of S x M x N doubles at ~4 TB/s
    // expressed in k-tile units (~1.3 us each)
    double t = waves * (kt + 2.0);
    if (S > 1) t += (double)S * g.M * g.N * 16.0 / 4e12 / 1.3e-6 + 2.0;
    if (t < best * 0.999) {
      best = t;
      p.splits = S;
      p.kt_per = kt;
    }
  }
  p.tiles = tiles;
  return p;
}

long long gemm_tma_workspace(const GemmArgs& g) {
  const TmaGemmPlan p = gemm_tma_plan(g);
  return p.splits > 1 ? (long long)p.splits * g.M * g.N : 0;
}

bool gemm_tma(const GemmArgs& g, cudaStream_t s, double* ws, long long ws_doubles) {
  if (!gemm_tma_eligible(g)) return false;
  const TmaGemmPlan p = gemm_tma_plan(g);
  if (p.splits > 1 && (ws == nullptr || ws_doubles < (long long)p.splits * g.M * g.N)) return false;
  static PerDevice<bool> attr_dev(false);
  bool& attr = attr_dev();
  if (!attr) {
    QTT_CUDA(cudaFuncSetAttribute(tma_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TC::SMEM));
    attr = true;
  }
  TmaGemmArgs a;
  make_tensor_map_2d(&a.ma, g.A, g.M, g.K, g.a_rs, TC::BM);
  make_tensor_map_2d(&a.mb, g.B, g.N, g.K, g.b_cs, TC::BN);
  a.M = g.M;
  a.N = g.N;
  a.K = g.K;
  a.tn = cdiv(g.N, TC::BN);
  a.tiles = p.tiles;
  a.splits = p.splits;
  a.kt_per = p.kt_per;
  a.C = g.C;
  a.ldc = g.c_rs;
  a.alpha = g.alpha;
  a.beta = g.beta;
  a.ws = ws;
  const int items = p.tiles * p.splits;
  const int grid = std::min(items, kSMs * kPerSM);
  tma_gemm_kernel<<<grid, TC::NT, TC::SMEM, s>>>(a);
  QTT_CHECK_LAUNCH();
  if (p.splits > 1) {
    const long long total = (long long)g.M * g.N;
    tma_splitk_reduce<<<(int)std::min<long long>(cdiv(total, 256), 4 * kSMs), 256, 0, s>>>(
        ws, p.splits, g.M, g.N, g.C, g.c_rs, g.alpha, g.beta);
    QTT_CHECK_LAUNCH();
  }
  return true;
}

}  // namespace qtt
