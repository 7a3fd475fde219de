// Runtime-shaped variant of the TMA tile engine (tma_tile.cuh): the CTA tile is a
// runtime grid of wm x wn warps, each owning a fixed 32 x 56 warp tile (4 x 7 DMMA
// fragments: 28 independent DMMAs per 11 fragment loads), so one kernel can match its tile height to the problem (e.g. M/148
// rows per CTA for a one-wave GEMM) instead of rounding the tile count up to a
// second partial wave.  TMA boxes (16-double K slices, 128B swizzle) carry the
// runtime tile height/width in their tensor maps.
#pragma once
#include "tma_tile.cuh"

namespace qtt {
namespace tmart {

constexpr int MI = 4, NI = 7;          // warp tile 32 x 56
constexpr int WROWS = 8 * MI, WCOLS = 8 * NI;
constexpr int STAGES = 4;

struct Shape {
  int wm, wn;  // CTA tile = (32*wm) x (56*wn); warps >= wm*wn idle in the GEMM
};
__host__ __device__ inline int shape_bm(Shape s) { return WROWS * s.wm; }
__host__ __device__ inline int shape_bn(Shape s) { return WCOLS * s.wn; }
__host__ __device__ inline int stage_bytes(Shape s) { return (shape_bm(s) + shape_bn(s)) * 128; }

struct Ring {
  unsigned char* base;  // 1024-aligned
  uint64_t* full;
  uint64_t* empty;
  unsigned uses;
  int stride;  // bytes per stage (multiple of 1024, >= every shape used)
};

__device__ __forceinline__ Ring ring_init(void* smem_raw, int stride) {
  Ring r;
  r.full = reinterpret_cast<uint64_t*>(smem_raw);
  r.empty = r.full + STAGES;
  uintptr_t p = reinterpret_cast<uintptr_t>(smem_raw) + 64;
  p = (p + 1023) & ~uintptr_t(1023);
  r.base = reinterpret_cast<unsigned char*>(p);
  r.uses = 0;
  r.stride = stride;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tma::mbar_init(&r.full[s], 1);
      tma::mbar_init(&r.empty[s], blockDim.x / 32);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  return r;
}

__device__ __forceinline__ void issue(Ring& r, unsigned slot, const tma::Item& it, int kt, Shape sh) {
  const int s = slot % STAGES;
  const unsigned f = slot / STAGES;
  if (f > 0) tma::mbar_wait(&r.empty[s], (f - 1) & 1u);
  unsigned char* st = r.base + (size_t)s * r.stride;
  tma::mbar_expect_tx(&r.full[s], stage_bytes(sh));
  tma::load_2d(st, it.ma, kt * 16, it.m0, &r.full[s]);
  tma::load_2d(st + shape_bm(sh) * 128, it.mb, kt * 16, it.n0, &r.full[s]);
}

__device__ __forceinline__ void compute(const Ring& r, unsigned slot, double (&acc)[MI][NI][2], Shape sh,
                                        int wm0, int wn0) {
  const int s = slot % STAGES;
  const unsigned sA = tma::smem_u32(r.base) + s * r.stride;
  const unsigned sB = sA + shape_bm(sh) * 128;
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 16; ks += 4) {
    const int off = tma::swz_off(ks >> 2, lr, lc);
    double af[MI], bf[NI];
#pragma unroll
    for (int i = 0; i < MI; ++i) af[i] = tma::lds64(sA + ((wm0 + i * 8 + lr) * 16 + off) * 8);
#pragma unroll
    for (int j = 0; j < NI; ++j) bf[j] = tma::lds64(sB + ((wn0 + j * 8 + lr) * 16 + off) * 8);
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) tile::dmma(acc[i][j], af[i], bf[j]);
  }
}

__device__ __forceinline__ void zero(double (&acc)[MI][NI][2]) {
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// Stream the k-tiles of items get(0..n-1) (all of shape sh) through the ring;
// epi(item, acc) after each item's last k-tile (called by every thread; idle warps
// hold zeros).  Thread 0 produces; consumers release stages on the empty barriers.
template <class Get, class Epi>
__device__ __forceinline__ void stream(Ring& r, Shape sh, int n_items, Get get, Epi epi) {
  if (n_items <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool active = warp < sh.wm * sh.wn;
  const int wm0 = (warp % sh.wm) * WROWS, wn0 = (warp / sh.wm) * WCOLS;
  int pi = 0, pk = 0;
  tma::Item P;
  const unsigned first = r.uses;
  unsigned produced = first;
  if (threadIdx.x == 0) {
    tma::fence_proxy_async();  // earlier generic-proxy use of the ring's shared memory
    P = get(0);
    pk = P.kb;
    for (int s = 0; s < STAGES - 1 && pi < n_items; ++s) {
      issue(r, produced++, P, pk, sh);
      if (++pk >= P.ke && ++pi < n_items) {
        P = get(pi);
        pk = P.kb;
      }
    }
  }
  __syncwarp();
  int ci = 0;
  tma::Item Cur = get(0);
  int ck = Cur.kb;
  double acc[MI][NI][2];
  zero(acc);
  unsigned slot = first;
  while (ci < n_items) {
    if (threadIdx.x == 0 && pi < n_items) {
      issue(r, produced++, P, pk, sh);
      if (++pk >= P.ke && ++pi < n_items) {
        P = get(pi);
        pk = P.kb;
      }
    }
    __syncwarp();
    tma::mbar_wait(&r.full[slot % STAGES], (slot / STAGES) & 1u);
    if (active) compute(r, slot, acc, sh, wm0, wn0);
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&r.empty[slot % STAGES]);
    ++slot;
    if (++ck >= Cur.ke) {
      epi(Cur, acc);
      zero(acc);
      if (++ci < n_items) {
        Cur = get(ci);
        ck = Cur.kb;
      }
    }
  }
  __syncthreads();
  r.uses = slot;
}

// Store this warp's part of a tile row by row (rowptr(row) -> destination of column 0).
template <class RowPtr>
__device__ __forceinline__ void store_rows(Shape sh, int m0, int n0, int M, int N, const double (&acc)[MI][NI][2],
                                          RowPtr&& rowptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= sh.wm * sh.wn) return;
  const int wm0 = (warp % sh.wm) * WROWS, wn0 = (warp / sh.wm) * WCOLS;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int row = m0 + wm0 + i * 8 + lr;
    if (row >= M) continue;
    double* dst = rowptr(row);
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int col = n0 + wn0 + j * 8 + lc * 2;
      if (col + 1 < N) {
        dst[col] = acc[i][j][0];
        dst[col + 1] = acc[i][j][1];
      } else if (col < N) {
        dst[col] = acc[i][j][0];
      }
    }
  }
}

}  // namespace tmart
}  // namespace qtt
