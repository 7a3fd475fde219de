// Device-side FP64 DMMA tile engine shared by the standalone GEMM kernel (gemm.cu)
// and the persistent fused kernels (cg_fused.cu): one CTA computes one BM x BN
// output tile over a K range, operands streamed global -> shared memory with
// cp.async in a STAGES-deep ring, fragments fed to mma.sync.m8n8k4.f64 (DMMA).
#pragma once
#include "gemm.cuh"

namespace qtt {
namespace tile {

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

template <int BM_, int BN_, int BK_, int WARPS_M_, int WARPS_N_, int STAGES_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int STAGES = STAGES_;
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
template <int BK, int BX>
__device__ __forceinline__ void tile_coord(int e, bool x_contig, int& kk, int& xx) {
  if (x_contig) {
    xx = e % BX;
    kk = e / BX;
  } else {
    int kq = e & 3, xq = (e >> 2) & 3, blk = e >> 4;
    kk = (blk % (BK / 4)) * 4 + kq;
    xx = (blk / (BK / 4)) * 4 + xq;
  }
}

// Operand views of one (batch) problem.
struct Operands {
  const double* A;
  long long a_rs, a_cs;
  const double* B;
  long long b_rs, b_cs;
  int M, N, K;
};

// acc += op(A)[m0:m0+BM, kt_begin*BK : kt_end*BK] @ op(B)[..., n0:n0+BN]
// smem: C::SMEM bytes.  All threads of the CTA must call it (contains barriers).
template <class C>
__device__ __forceinline__ void mma_tile(const Operands& o, int m0, int n0, int kt_begin, int kt_end,
                                         double* smem, double (&acc)[C::MI][C::NI][2]) {
  constexpr int NT = C::NT, LDA = C::LDA, LDB = C::LDB, BK = C::BK, BM = C::BM, BN = C::BN;
  constexpr int STAGES = C::STAGES;
  double* sA = smem;
  double* sB = smem + STAGES * BK * LDA;
  const bool a_mc = (o.a_rs == 1);
  const bool b_nc = (o.b_cs == 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp % C::WARPS_M) * C::WTM;
  const int wn0 = (warp / C::WARPS_M) * C::WTN;
  const int lr = lane >> 2, lc = lane & 3;

  auto load_tile = [&](int kt, int stage) {
    const int k0 = kt * BK;
    double* dA = sA + stage * BK * LDA;
    double* dB = sB + stage * BK * LDB;
#pragma unroll
    for (int i = 0; i < (BM * BK) / NT; ++i) {
      int kk, mm;
      tile_coord<BK, BM>(threadIdx.x + i * NT, a_mc, kk, mm);
      const int gm = m0 + mm, gk = k0 + kk;
      const bool ok = gm < o.M && gk < o.K;
      const double* src = ok ? o.A + (long long)gm * o.a_rs + (long long)gk * o.a_cs : o.A;
      cp_async8(dA + kk * LDA + mm, src, ok);
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / NT; ++i) {
      int kk, nn;
      tile_coord<BK, BN>(threadIdx.x + i * NT, b_nc, kk, nn);
      const int gn = n0 + nn, gk = k0 + kk;
      const bool ok = gn < o.N && gk < o.K;
      const double* src = ok ? o.B + (long long)gk * o.b_rs + (long long)gn * o.b_cs : o.B;
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
      double af[C::MI], bf[C::NI];
#pragma unroll
      for (int i = 0; i < C::MI; ++i) af[i] = cA[(ks + lc) * LDA + wm0 + i * 8 + lr];
#pragma unroll
      for (int j = 0; j < C::NI; ++j) bf[j] = cB[(ks + lc) * LDB + wn0 + j * 8 + lr];
#pragma unroll
      for (int i = 0; i < C::MI; ++i)
#pragma unroll
        for (int j = 0; j < C::NI; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // the ring may be reused by the caller's next tile
}

template <class C>
__device__ __forceinline__ void zero_acc_impl(double (&acc)[C::MI][C::NI][2]) {
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// One unit of a CTA's work list: output tile (m0, n0) of operands o over k-tiles [kb, ke).
struct TileItem {
  Operands o;
  int m0, n0, kb, ke;
};

// Issue the cp.async copies of k-tile kt of item it into ring stage `stage`.
template <class C>
__device__ __forceinline__ void load_stage(const TileItem& it, int kt, int stage, double* smem) {
  constexpr int NT = C::NT, LDA = C::LDA, LDB = C::LDB, BK = C::BK, BM = C::BM, BN = C::BN;
  double* dA = smem + stage * BK * LDA;
  double* dB = smem + C::STAGES * BK * LDA + stage * BK * LDB;
  const Operands& o = it.o;
  const bool a_mc = (o.a_rs == 1), b_nc = (o.b_cs == 1);
  const int k0 = kt * BK;
#pragma unroll
  for (int i = 0; i < (BM * BK) / NT; ++i) {
    int kk, mm;
    tile_coord<BK, BM>(threadIdx.x + i * NT, a_mc, kk, mm);
    const int gm = it.m0 + mm, gk = k0 + kk;
    const bool ok = gm < o.M && gk < o.K;
    const double* src = ok ? o.A + (long long)gm * o.a_rs + (long long)gk * o.a_cs : o.A;
    cp_async8(dA + kk * LDA + mm, src, ok);
  }
#pragma unroll
  for (int i = 0; i < (BN * BK) / NT; ++i) {
    int kk, nn;
    tile_coord<BK, BN>(threadIdx.x + i * NT, b_nc, kk, nn);
    const int gn = it.n0 + nn, gk = k0 + kk;
    const bool ok = gn < o.N && gk < o.K;
    const double* src = ok ? o.B + (long long)gk * o.b_rs + (long long)gn * o.b_cs : o.B;
    cp_async8(dB + kk * LDB + nn, src, ok);
  }
}

template <class C>
__device__ __forceinline__ void compute_stage(int stage, const double* smem, double (&acc)[C::MI][C::NI][2]) {
  constexpr int LDA = C::LDA, LDB = C::LDB, BK = C::BK;
  const double* cA = smem + stage * BK * LDA;
  const double* cB = smem + C::STAGES * BK * LDA + stage * BK * LDB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp % C::WARPS_M) * C::WTM;
  const int wn0 = (warp / C::WARPS_M) * C::WTN;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int ks = 0; ks < BK; ks += 4) {
    double af[C::MI], bf[C::NI];
#pragma unroll
    for (int i = 0; i < C::MI; ++i) af[i] = cA[(ks + lc) * LDA + wm0 + i * 8 + lr];
#pragma unroll
    for (int j = 0; j < C::NI; ++j) bf[j] = cB[(ks + lc) * LDB + wn0 + j * 8 + lr];
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) dmma(acc[i][j], af[i], bf[j]);
  }
}

// Persistent work stream: all k-tiles of the CTA's items (get(0..n-1)) flow through
// ONE cp.async ring, so the loads of item i+1 are in flight while item i finishes and
// its epilogue epi(item, acc) stores -- no pipeline refill bubble per tile.
template <class C, class Get, class Epi>
__device__ __forceinline__ void mma_stream(int n_items, Get get, Epi epi, double* smem) {
  if (n_items <= 0) return;
  constexpr int STAGES = C::STAGES;
  int li = 0;
  TileItem L = get(0);
  int lk = L.kb;
  auto next_load = [&](int stage) {
    if (li >= n_items) return;
    load_stage<C>(L, lk, stage, smem);
    if (++lk >= L.ke) {
      if (++li < n_items) {
        L = get(li);
        lk = L.kb;
      }
    }
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    next_load(s);
    cp_async_commit();
  }
  int ci = 0;
  TileItem Cur = get(0);
  int ck = Cur.kb;
  double acc[C::MI][C::NI][2];
  zero_acc_impl<C>(acc);
  for (int step = 0; ci < n_items; ++step) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    next_load((step + STAGES - 1) % STAGES);
    cp_async_commit();
    compute_stage<C>(step % STAGES, smem, acc);
    if (++ck >= Cur.ke) {
      epi(Cur, acc);
      zero_acc_impl<C>(acc);
      if (++ci < n_items) {
        Cur = get(ci);
        ck = Cur.kb;
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

// Visit every accumulator element: f(row, col, value) for in-range entries.
template <class C, class F>
__device__ __forceinline__ void for_each_acc(int m0, int n0, int M, int N, const double (&acc)[C::MI][C::NI][2],
                                             F&& f) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp % C::WARPS_M) * C::WTM;
  const int wn0 = (warp / C::WARPS_M) * C::WTN;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) {
      const int row = m0 + wm0 + i * 8 + lr;
      const int col = n0 + wn0 + j * 8 + lc * 2;
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (row < M && col + t < N) f(row, col + t, acc[i][j][t]);
    }
}

template <class C>
__device__ __forceinline__ void zero_acc(double (&acc)[C::MI][C::NI][2]) {
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

}  // namespace tile
}  // namespace qtt
