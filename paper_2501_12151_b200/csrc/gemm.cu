// FP64 DMMA GEMM (see gemm.cuh for the operand convention); the tile engine
// itself lives in dmma_tile.cuh and is shared with the persistent fused kernels.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "dmma_tile.cuh"
#include "gemm.cuh"
#include "gemm_tma.cuh"

namespace qtt {
namespace {

template <class C>
__global__ void __launch_bounds__(C::NT)
    dgemm_kernel(GemmArgs g, int splits, int kt_per_split, double* __restrict__ ws) {
  extern __shared__ double smem[];
  if (g.skip != nullptr && *g.skip != 0) return;
  if (g.lower_only && (int)(blockIdx.x * C::BN) >= (int)(blockIdx.y * C::BM + C::BM)) return;
  int z = blockIdx.z;
  const int split = z % splits;
  z /= splits;
  const int b1 = z % g.batch1;
  const int b2 = z / g.batch1;
  tile::Operands o{g.A + b1 * g.a_bs1 + b2 * g.a_bs2, g.a_rs, g.a_cs,
                   g.B + b1 * g.b_bs1 + b2 * g.b_bs2, g.b_rs, g.b_cs, g.M, g.N, g.K};
  const int m0 = blockIdx.y * C::BM, n0 = blockIdx.x * C::BN;
  const int ktiles = (g.K + C::BK - 1) / C::BK;
  const int kt_begin = split * kt_per_split;
  const int kt_end = min(ktiles, kt_begin + kt_per_split);
  double acc[C::MI][C::NI][2];
  tile::zero_acc<C>(acc);
  tile::mma_tile<C>(o, m0, n0, kt_begin, kt_end, smem, acc);
  if (splits > 1) {
    double* W = ws + (long long)split * g.M * g.N;
    const int N = g.N;
    tile::for_each_acc<C>(m0, n0, g.M, g.N, acc, [&](int r, int c, double v) { W[(long long)r * N + c] = v; });
    return;
  }
  double* Cp = g.C + b1 * g.c_bs1 + b2 * g.c_bs2;
  const double alpha = g.alpha, beta = g.beta;
  const bool lower = g.lower_only;
  tile::for_each_acc<C>(m0, n0, g.M, g.N, acc, [&](int r, int c, double v) {
    if (lower && c > r) return;
    double* p = Cp + (long long)r * g.c_rs + (long long)c * g.c_cs;
    double out = alpha * v;
    if (beta != 0.0) out = fma(beta, *p, out);
    *p = out;
  });
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

template <class C>
void launch(const GemmArgs& g, int splits, int kt_per, double* ws, cudaStream_t s) {
  static PerDevice<bool> attr_dev(false);  // per-instantiation, set once per device
  bool& attr_set = attr_dev();
  if (!attr_set) {
    QTT_CUDA(cudaFuncSetAttribute(dgemm_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)C::SMEM));
    attr_set = true;
  }
  long long zb = (long long)g.batch1 * g.batch2 * splits;
  if (zb > 65535) throw Error(QTT_ERR_ARG, "gemm: batch too large for grid.z");
  dim3 grid(cdiv(g.N, C::BN), cdiv(g.M, C::BM), (unsigned)zb);
  dgemm_kernel<C><<<grid, C::NT, C::SMEM, s>>>(g, splits, kt_per, ws);
  QTT_CHECK_LAUNCH();
}

using Cfg64 = tile::Cfg<64, 64, 16, 2, 2, 3>;
using Cfg32 = tile::Cfg<32, 32, 16, 2, 2, 4>;
using Cfg128 = tile::Cfg<128, 64, 16, 4, 2, 3>;
using Cfg128x128 = tile::Cfg<128, 128, 16, 4, 2, 3>;

constexpr int kSMs = 148;

struct Plan {
  int cfg;      // 0: 64x64, 1: 32x32, 2: 128x64, 3: 128x128
  int splits;
  int kt_per;
};

// Pick the tile shape and split-K count with the smallest modelled time: full waves of
// CTAs over the 148 SMs x (tile area x k-tiles) / relative per-SM DMMA efficiency of the
// tile (bigger warp tiles issue fewer shared loads per DMMA and hide more latency), plus
// the split-K partial traffic.  Split-K only for unbatched products short of a full wave.
Plan plan_for(const GemmArgs& g) {
  const long long batch = (long long)g.batch1 * g.batch2;
  const int ktiles = cdiv(g.K, 16);
  struct Cand { int cfg, bm, bn; double eff; int per_sm; };
  const Cand cands[] = {{3, 128, 128, 0.8, 1}, {2, 128, 64, 0.9, 2}, {0, 64, 64, 0.62, 3}, {1, 32, 32, 0.3, 4}};
  Plan best{0, 1, ktiles};
  double best_t = 1e300;
  for (const Cand& c : cands) {
    if (c.cfg == 3 && (g.M < 256 || g.N < 256)) continue;
    if (c.cfg == 2 && g.M < 96) continue;
    if (c.cfg != 1 && (g.M <= 40 || g.N <= 40)) continue;
    const long long tiles = (long long)cdiv(g.M, c.bm) * cdiv(g.N, c.bn) * batch;
    int splits = 1;
    if (batch == 1 && tiles < (long long)kSMs * c.per_sm && ktiles >= 16) {
      const int want = (int)std::min<long long>(std::max<long long>(1, (long long)kSMs * c.per_sm / tiles),
                                                ktiles / 8);
      splits = std::max(1, want);
    }
    const int kt_per = cdiv(ktiles, splits);
    splits = cdiv(ktiles, kt_per);
    const long long ctas = tiles * splits;
    const double waves = std::ceil((double)ctas / ((double)kSMs * c.per_sm));
    // time units: one DMMA-efficient 128x128x16 tile step = 1
    double t = waves * c.per_sm * ((double)c.bm * c.bn / (128.0 * 128.0)) * kt_per / c.eff;
    if (splits > 1) t += (double)splits * g.M * g.N * 16.0 / (128.0 * 128.0 * 16.0 * 2.0 * kSMs) * 4.0 + 2.0;
    if (t < best_t * 0.999) {
      best_t = t;
      best = Plan{c.cfg, splits, kt_per};
    }
  }
  if (const char* e = std::getenv("QTT_GEMM_CFG")) best.cfg = std::atoi(e);  // tuning override
  return best;
}

}  // namespace

static bool tma_path_on() {
  static const bool on = !(std::getenv("QTT_GEMM_TMA") && std::atoi(std::getenv("QTT_GEMM_TMA")) == 0);
  return on;
}

long long gemm_workspace_hint(const GemmArgs& g) {
  if (tma_path_on() && gemm_tma_eligible(g)) return gemm_tma_workspace(g);
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
  if (tma_path_on() && gemm_tma(g, s, ws, ws_doubles)) return;
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
    case 1: launch<Cfg32>(g, p.splits, p.kt_per, ws, s); break;
    case 2: launch<Cfg128>(g, p.splits, p.kt_per, ws, s); break;
    case 3: launch<Cfg128x128>(g, p.splits, p.kt_per, ws, s); break;
    default: launch<Cfg64>(g, p.splits, p.kt_per, ws, s); break;
  }
  if (p.splits > 1) {
    const long long total = (long long)g.M * g.N;
    int blocks = (int)std::min<long long>(cdiv(total, 256), 4 * kSMs);
    splitk_reduce<<<blocks, 256, 0, s>>>(ws, p.splits, g.M, g.N, g.C, g.c_rs, g.c_cs, g.alpha, g.beta, g.skip);
    QTT_CHECK_LAUNCH();
  }
}

}  // namespace qtt
