// Fragment-balanced TMA/DMMA engine for one-wave GEMM phases of a persistent kernel.
//
// The small local-system GEMMs of the AMEn sweep (e.g. 10400 x 100 x 200 at rank
// 100) are too small for fixed CTA tiles: rounding the tile count to the 148 SMs,
// and the warp count of a tile to the 4 schedulers per SM, idles up to half of the
// DMMA pipes (tools/tile_bench.cu).  Here each CTA gets an output REGION sized to
// its exact share of the work (a run of 8-row fragment rows, all columns, or a
// column block), and inside the region the 8x8 DMMA fragments are dealt out to the
// 12 warps (3 per scheduler) in equal contiguous runs (row-major), so every
// scheduler issues the same number of DMMAs.  A warp keeps up to MAXF fragment
// accumulators; when its run spans at most 2 fragment rows the A fragments are
// loaded once per row and picked with a predicated select.
//
// Operands are K-contiguous (C = A . B^T); per k-tile one TMA box of A rows and one
// of B rows (16 doubles of K each, 128B swizzle) land in a 4-stage ring guarded by
// full/empty mbarriers; thread 0 produces.
#pragma once
#include "tma_tile.cuh"

namespace qtt {
namespace tmafb {

constexpr int MAXF = 16;   // fragments per warp (largest instantiation)
constexpr int NWARP = 12;  // consumer warps per CTA: 3 per scheduler
constexpr int STAGES = 4;      // ring depth (deeper rings only delayed the first k-tile: the
                               // prologue burst of every CTA queues behind the others in L2)
constexpr int MAX_STAGES = STAGES;
constexpr int HEADER = 256;    // mbarriers (full + empty per stage) before the ring

// One unit of work: output rows [m0, m0+mrows) x cols [n0, n0+ncols), k-tiles [kb, ke).
struct Region {
  int m0, mrows, n0, ncols, kb, ke;
};

struct Ring {
  unsigned char* base;  // 1024-aligned
  uint64_t* full;
  uint64_t* empty;
  unsigned uses;
  int stride;                 // bytes per stage (multiple of 1024)
  int nst;                    // stages
  unsigned long long* dbg;    // optional: CTA 0 stream timeline accumulators (4 per stream slot)
  int dbg_slot;
};

__device__ __forceinline__ unsigned long long fb_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ Ring ring_init(void* smem_raw, int stride, int nst) {
  Ring r;
  r.full = reinterpret_cast<uint64_t*>(smem_raw);
  r.empty = r.full + MAX_STAGES;
  uintptr_t p = reinterpret_cast<uintptr_t>(smem_raw) + HEADER;
  p = (p + 1023) & ~uintptr_t(1023);
  r.base = reinterpret_cast<unsigned char*>(p);
  r.uses = 0;
  r.stride = stride;
  r.nst = nst;
  r.dbg = nullptr;
  r.dbg_slot = 0;
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

// Operand boxes of a phase: box_a rows of A (at y = m0), box_b rows of B (at y = n0).
struct Boxes {
  const CUtensorMap* ma;
  const CUtensorMap* mb;
  int box_a, box_b;
};

__device__ __forceinline__ void issue(Ring& r, unsigned slot, const Boxes& bx, const Region& g, int kt) {
  const int s = slot % STAGES;
  const unsigned f = slot / STAGES;
  if (f > 0) tma::mbar_wait(&r.empty[s], (f - 1) & 1u);
  unsigned char* st = r.base + (size_t)s * r.stride;
  tma::mbar_expect_tx(&r.full[s], (bx.box_a + bx.box_b) * 128);
  tma::load_2d(st, bx.ma, kt * 16, g.m0, &r.full[s]);
  tma::load_2d(st + bx.box_a * 128, bx.mb, kt * 16, g.n0, &r.full[s]);
}

// This warp's fragment run inside a region: fragments g0 .. g0+NF-1 of the
// FM x FN fragment grid (row-major; every warp's run is NF long -- fragments past
// the region compute on valid shared memory and are dropped at the store).  With
// DEDUPE the run spans at most 2 fragment rows: row i0 up to fragment t1-1, then
// row i0+1.
template <int NF>
struct Frags {
  int t1;          // first fragment of the second row (NF if none)
  unsigned valid;  // bit f: fragment f inside the region
  int boff[NF];    // B fragment row offset in the stage (doubles, incl. lane row)
  int aoff[NF];    // A fragment row offset (doubles, incl. lane row)
};

template <int NF>
__device__ __forceinline__ void frags_for(const Region& g, Frags<NF>& fr) {
  const int FN = (g.ncols + 7) >> 3, FM = (g.mrows + 7) >> 3;
  const int F = FM * FN;
  const int warp = threadIdx.x >> 5, lr = (threadIdx.x & 31) >> 2;
  const int g0 = warp * NF;
  // a warp past the region keeps row/col 0 for its (dropped) fragments: all of its
  // shared-memory reads stay inside the stage
  const int i0 = g0 < F ? g0 / FN : 0;
  int i = i0, j = g0 < F ? g0 - i0 * FN : 0;
  fr.valid = 0u;
  fr.t1 = NF;
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const bool ok = g0 + f < F;
    if (ok) fr.valid |= 1u << f;
    if (i != i0 && fr.t1 == NF) fr.t1 = f;
    const int ii = ok ? i : i0, jj = ok ? j : 0;  // dropped fragments read row/col 0 of the run
    fr.aoff[f] = (ii * 8 + lr) * 16;
    fr.boff[f] = (jj * 8 + lr) * 16;
    if (++j == FN) {
      j = 0;
      ++i;
    }
  }
}

template <int NF, bool DEDUPE>
__device__ __forceinline__ void compute(const Ring& r, unsigned slot, const Boxes& bx, const Frags<NF>& fr,
                                        double (&acc)[NF][2]) {
  const int s = slot % STAGES;
  const unsigned sA = tma::smem_u32(r.base) + s * r.stride;
  const unsigned sB = sA + bx.box_a * 128;
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 16; ks += 4) {
    const int off = tma::swz_off(ks >> 2, lr, lc);
    double b[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) b[f] = tma::lds64(sB + (fr.boff[f] + off) * 8);
    if constexpr (DEDUPE) {
      const double x0 = tma::lds64(sA + (fr.aoff[0] + off) * 8);
      const double x1 = tma::lds64(sA + (fr.aoff[0] + 128 + off) * 8);
#pragma unroll
      for (int f = 0; f < NF; ++f) tile::dmma(acc[f], f < fr.t1 ? x0 : x1, b[f]);
    } else {
#pragma unroll
      for (int f = 0; f < NF; ++f) tile::dmma(acc[f], tma::lds64(sA + (fr.aoff[f] + off) * 8), b[f]);
    }
  }
}

// Stream regions get(0..n-1) through the ring; epi(region, frags, acc) after each
// region's last k-tile (all threads call it).
template <int NF, bool DEDUPE, class Get, class Epi>
__device__ __forceinline__ void stream(Ring& r, const Boxes& bx, int n, Get get, Epi epi) {
  if (n <= 0) return;
  const int lane = threadIdx.x & 31;
  const bool tl = r.dbg != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  const unsigned long long t_start = tl ? fb_clock() : 0;
  int pi = 0, pk = 0;
  Region P;
  const unsigned first = r.uses;
  unsigned produced = first;
  if (threadIdx.x == 0) {
    tma::fence_proxy_async();  // earlier generic-proxy use of the ring's shared memory
    P = get(0);
    pk = P.kb;
    for (int s = 0; s < STAGES - 1 && pi < n; ++s) {
      issue(r, produced++, bx, P, pk);
      if (++pk >= P.ke && ++pi < n) {
        P = get(pi);
        pk = P.kb;
      }
    }
  }
  __syncwarp();
  int ci = 0;
  Region Cur = get(0);
  int ck = Cur.kb;
  Frags<NF> fr;
  frags_for<NF>(Cur, fr);
  double acc[NF][2];
#pragma unroll
  for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
  unsigned slot = first;
  while (ci < n) {
    if (threadIdx.x == 0 && pi < n) {
      issue(r, produced++, bx, P, pk);
      if (++pk >= P.ke && ++pi < n) {
        P = get(pi);
        pk = P.kb;
      }
    }
    __syncwarp();
    const unsigned st = slot % STAGES;
    tma::mbar_wait(&r.full[st], (slot / STAGES) & 1u);
    compute<NF, DEDUPE>(r, slot, bx, fr, acc);
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&r.empty[st]);
    ++slot;
    if (++ck >= Cur.ke) {
      if (tl) r.dbg[4 * r.dbg_slot + 1] += fb_clock() - t_start;
      epi(Cur, fr, acc);
      if (tl) r.dbg[4 * r.dbg_slot + 2] += fb_clock() - t_start;
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
      if (++ci < n) {
        Cur = get(ci);
        ck = Cur.kb;
        frags_for<NF>(Cur, fr);
      }
    }
  }
  __syncthreads();
  if (tl) r.dbg[4 * r.dbg_slot + 3] += fb_clock() - t_start;
  r.uses = slot;
}

// Store this warp's fragments of region g (limits M, N): rowptr(row) -> column 0 of row.
template <int NF, class RowPtr>
__device__ __forceinline__ void store(const Region& g, const Frags<NF>& fr, const double (&acc)[NF][2], int M,
                                     int N, RowPtr&& rowptr) {
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const int rlim = min(M, g.m0 + g.mrows), clim = min(N, g.n0 + g.ncols);
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    if (fr.valid & (1u << f)) {
      const int row = g.m0 + fr.aoff[f] / 16;
      const int col = g.n0 + (fr.boff[f] / 16 - lr) + lc * 2;
      if (row < rlim) {
        double* dst = rowptr(row);
        if (col + 1 < clim) {
          dst[col] = acc[f][0];
          dst[col + 1] = acc[f][1];
        } else if (col < clim) {
          dst[col] = acc[f][0];
        }
      }
    }
  }
}

// Fragments per warp for a region of F fragments (instantiated sizes).
__host__ __device__ inline int nf_for(int F) {
  const int per = (F + NWARP - 1) / NWARP;
  return per <= 4 ? 4 : per <= 6 ? 6 : per <= 8 ? 8 : per <= 10 ? 10 : per <= 12 ? 12 : 16;
}
// A warp run of nf fragments over rows of fn fragments spans at most 2 rows.
__host__ __device__ inline bool dedupe_ok(int nf, int fn) { return nf <= fn + 1; }

}  // namespace tmafb
}  // namespace qtt
