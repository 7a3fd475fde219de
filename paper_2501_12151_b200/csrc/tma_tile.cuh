// TMA-fed FP64 DMMA tile engine (sm_100a).  Both operands are K-contiguous in
// global memory (C = A . B^T with A [M][K], B [N][K]); one thread issues
// cp.async.bulk.tensor copies of 16-double (128-byte) K slices per row into a
// STAGES-deep shared-memory ring with the hardware 128-byte swizzle, completion
// tracked by one mbarrier per stage.  The 8 consumer warps read DMMA fragments
// straight from the swizzled layout (conflict-free: lane row r reads 16-byte chunk
// (k/2) ^ (r%8)), so the main loop is DMMA + LDS only -- no per-element address
// arithmetic, which is what held the cp.async engine (dmma_tile.cuh) to ~60% of the
// DMMA pipe (tools/tile_bench.cu).
#pragma once
#include <cuda.h>

#include <cstdint>

#include "dmma_tile.cuh"

namespace qtt {
namespace tma {

template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int STAGES_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = 16, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int STAGES = STAGES_;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MI = WTM / 8, NI = WTN / 8;
  static constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // mbarriers (64 B) + alignment slack to 1024 B (128B swizzle) + the ring
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 64 + 1024;
  static_assert(WTM % 8 == 0 && WTN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert(BM % 8 == 0 && BN % 8 == 0 && BM <= 256 && BN <= 256, "TMA box rows");
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// 8-byte shared-memory load at a 32-bit shared address.  The ring base is realigned
// at run time through integer arithmetic, which loses the pointer's address space:
// plain C++ loads through it compile to generic LD with 64-bit address math per
// fragment (measured: half the DMMA rate); explicit ld.shared keeps LDS + 32-bit adds.
__device__ __forceinline__ double lds64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 2D tensor copy: box at (x = K offset, y = row offset) -> dst, completing on bar.
__device__ __forceinline__ void load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(map) : "memory");
}

// Column (in doubles) of the 128B-swizzled 16-double row that lane (lr, lc) reads in
// k-step s (0..3) of a k-tile.  The k order inside a k-tile is free (it is summed
// over), so k-step s takes the two 16-byte chunks s and s+4: lanes lc = 0,1 read
// chunk s, lanes 2,3 chunk s+4.  Rows lr and lr^4 then share physical chunks only
// across half-warps, so every half-warp's 16 8-byte loads hit 32 distinct banks
// (with k-steps over consecutive chunk pairs, rows lr and lr^1 collided: 2-way
// conflicts on half of all fragment loads, tools/tile_bench.cu + ncu).
__device__ __forceinline__ int swz_off(int s, int lr, int lc) {
  const int chunk = (s + ((lc >> 1) << 2)) ^ lr;
  return (chunk << 1) | (lc & 1);
}

// One unit of work: output tile (m0, n0) of A.B^T over k-tiles [kb, ke).
struct Item {
  const CUtensorMap* ma;
  const CUtensorMap* mb;
  int m0, n0, kb, ke;
};

// Ring state shared by consecutive streams of one CTA (phases of a persistent
// kernel, possibly with different tile shapes of the same STAGES): the mbarriers
// live at the front of shared memory and their phase bits continue across calls.
struct Ring {
  unsigned char* base;  // 1024-aligned
  uint64_t* full;       // TMA bytes landed (count 1 + tx)
  uint64_t* empty;      // every consumer warp done with the stage (count NT/32)
  unsigned uses;        // k-tiles consumed so far (all stages)
};

template <int STAGES>
__device__ __forceinline__ Ring ring_init(void* smem_raw) {
  static_assert(STAGES <= 4, "mbarrier area is 64 bytes (full + empty per stage)");
  Ring r;
  r.full = reinterpret_cast<uint64_t*>(smem_raw);
  r.empty = r.full + 4;
  uintptr_t p = reinterpret_cast<uintptr_t>(smem_raw) + 64;
  p = (p + 1023) & ~uintptr_t(1023);
  r.base = reinterpret_cast<unsigned char*>(p);
  r.uses = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&r.full[s], 1);
      mbar_init(&r.empty[s], blockDim.x / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  return r;
}

// Fill number f = slot / STAGES of stage slot % STAGES; from the second fill on, wait
// until every consumer warp released the stage's previous fill (empty barrier).
template <class C>
__device__ __forceinline__ void issue(Ring& r, unsigned slot, const Item& it, int kt) {
  const int s = slot % C::STAGES;
  const unsigned f = slot / C::STAGES;
  if (f > 0) mbar_wait(&r.empty[s], (f - 1) & 1u);
  unsigned char* st = r.base + (size_t)s * C::STAGE_BYTES;
  mbar_expect_tx(&r.full[s], C::STAGE_BYTES);
  load_2d(st, it.ma, kt * 16, it.m0, &r.full[s]);
  load_2d(st + C::A_BYTES, it.mb, kt * 16, it.n0, &r.full[s]);
}

template <class C>
__device__ __forceinline__ void compute(const Ring& r, unsigned slot, double (&acc)[C::MI][C::NI][2]) {
  const int s = slot % C::STAGES;
  const unsigned sA = smem_u32(r.base) + s * C::STAGE_BYTES;
  const unsigned sB = sA + C::A_BYTES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp % C::WARPS_M) * C::WTM;
  const int wn0 = (warp / C::WARPS_M) * C::WTN;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 16; ks += 4) {
    const int off = swz_off(ks >> 2, lr, lc);  // swizzled column of (row%8 == lr, k)
    double af[C::MI], bf[C::NI];
#pragma unroll
    for (int i = 0; i < C::MI; ++i) af[i] = lds64(sA + ((wm0 + i * 8 + lr) * 16 + off) * 8);
#pragma unroll
    for (int j = 0; j < C::NI; ++j) bf[j] = lds64(sB + ((wn0 + j * 8 + lr) * 16 + off) * 8);
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) tile::dmma(acc[i][j], af[i], bf[j]);
  }
}

template <class C>
__device__ __forceinline__ void zero(double (&acc)[C::MI][C::NI][2]) {
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// Stream the k-tiles of items get(0..n-1) through the ring; epi(item, acc) after
// the last k-tile of each item.  All threads must call it.  Thread 0 produces.
template <class C, class Get, class Epi>
__device__ __forceinline__ void stream(Ring& r, int n_items, Get get, Epi epi) {
  if (n_items <= 0) return;
  constexpr int S = C::STAGES;
  // producer cursor (thread 0 only)
  int pi = 0, pk = 0;
  Item P;
  const unsigned first = r.uses;
  unsigned produced = first;
  if (threadIdx.x == 0) {
    fence_proxy_async();  // earlier generic-proxy use of the ring's shared memory
    P = get(0);
    pk = P.kb;
    for (int s = 0; s < S - 1 && pi < n_items; ++s) {
      issue<C>(r, produced++, P, pk);
      if (++pk >= P.ke && ++pi < n_items) {
        P = get(pi);
        pk = P.kb;
      }
    }
  }
  __syncwarp();
  int ci = 0;
  Item Cur = get(0);
  int ck = Cur.kb;
  double acc[C::MI][C::NI][2];
  zero<C>(acc);
  unsigned slot = first;
  const int lane = threadIdx.x & 31;
  while (ci < n_items) {
    // refill the stage released one step ago (the producer waits on its empty
    // barrier; the other warps run ahead while their data is already resident)
    if (threadIdx.x == 0 && pi < n_items) {
      issue<C>(r, produced++, P, pk);
      if (++pk >= P.ke && ++pi < n_items) {
        P = get(pi);
        pk = P.kb;
      }
    }
    __syncwarp();  // reconverge warp 0 before the warp-synchronous DMMAs
    mbar_wait(&r.full[slot % S], (slot / S) & 1u);
    compute<C>(r, slot, acc);
    __syncwarp();
    if (lane == 0) mbar_arrive(&r.empty[slot % S]);
    ++slot;
    if (++ck >= Cur.ke) {
      epi(Cur, acc);
      zero<C>(acc);
      if (++ci < n_items) {
        Cur = get(ci);
        ck = Cur.kb;
      }
    }
  }
  __syncthreads();
  r.uses = slot;
}

// Visit every accumulator element: f(row, col, value) for in-range entries.
template <class C, class F>
__device__ __forceinline__ void for_each(int m0, int n0, int M, int N, const double (&acc)[C::MI][C::NI][2], F&& f) {
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

// Store the accumulator tile row by row: rowptr(row) gives the destination of
// column 0 of that (in-range) row; one call per row and fragment.
template <class C, class RowPtr>
__device__ __forceinline__ void store_rows(int m0, int n0, int M, int N, const double (&acc)[C::MI][C::NI][2],
                                          RowPtr&& rowptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp % C::WARPS_M) * C::WTM;
  const int wn0 = (warp / C::WARPS_M) * C::WTN;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int i = 0; i < C::MI; ++i) {
    const int row = m0 + wm0 + i * 8 + lr;
    if (row >= M) continue;
    double* dst = rowptr(row);
#pragma unroll
    for (int j = 0; j < C::NI; ++j) {
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

}  // namespace tma

// Host: 2D tensor map of a row-major [rows][cols] FP64 matrix with row stride
// ld (elements; ld*8 must be a multiple of 16), box = 16 columns x box_rows rows,
// 128-byte swizzle, zero fill out of bounds.  Throws on driver error.
void make_tensor_map_2d(CUtensorMap* map, const double* base, long long rows, long long cols, long long ld,
                        int box_rows);

}  // namespace qtt
