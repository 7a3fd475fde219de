// Pair-dealt TMA/DMMA engine for one-wave GEMM phases of a persistent kernel.
//
// The local-system GEMMs of the AMEn sweep (e.g. 6200 x 100 x 200 at x rank 100, operator
// rank 31) are too small for fixed CTA tiles: rounding to whole tiles, or even to whole
// 8-row fragment rows per CTA, idles a fifth of the DMMA pipe, and a warp that owns a plain
// run of 8x8 fragments loads one B fragment per DMMA (shared-memory port ~70% busy next to
// the DMMA pipe: the loop reached 64-73% of the DMMA issue rate, tools/tile_bench.cu).
//
// Here the output fragment grid (FM x FN fragments of 8x8) is cut into 2-row STRIPS, and the
// unit of work is a vertical PAIR of fragments (rows 2s, 2s+1 of one fragment column: one B
// fragment feeds two DMMAs).  Pairs are numbered strip by strip, column by column (an odd last
// fragment row forms horizontal pairs); a CTA owns a contiguous range of pairs -- its exact
// 1/G share of the whole grid -- and inside a region the pairs are dealt to the 12 warps in
// equal runs of NP.  A run of NP <= FN pairs touches at most two strips, so a warp loads at
// most 4 A fragments and NP B fragments for its 2 NP DMMAs per k-step.
//
// Operands are K-contiguous (C = A . B^T); per k-tile one TMA box of A rows (the strips the
// region touches) and one of B rows (16 doubles of K each, 128B swizzle) land in a ring of
// run-time depth guarded by full/empty mbarriers; thread 0 produces.
#pragma once
#include "tma_tile.cuh"

namespace qtt {
namespace tmapr {

constexpr int MAXNP = 8;        // pairs per warp (largest instantiation: 16 accumulator fragments)
constexpr int NWARP = 12;       // consumer warps per CTA: 3 per scheduler
constexpr int MAX_STAGES = 12;  // deepest ring (run-time depth: Ring::nst)
constexpr int HEADER = 256;     // mbarriers (full + empty per stage) before the ring

// One unit of work: pairs [pb, pe) of the fragment grid whose fragment (0, 0) is the output
// block at (m0, n0), FM x FN fragments, over k-tiles [kb, ke) visited in the rotated order
// kb+rot, .., ke-1, kb, .., kb+rot-1 (0 <= rot < ke - kb).  pb >= pe: nothing to do.
struct Region {
  int m0, n0, FM, FN, pb, pe, kb, ke, rot;
};

// pairs of an FM x FN fragment grid
__host__ __device__ inline int pairs_of(int FM, int FN) { return (FM >> 1) * FN + ((FM & 1) ? (FN + 1) / 2 : 0); }
// strip of pair p
__host__ __device__ inline int strip_of(int p, int FM, int FN) {
  const int FS = FM >> 1;
  return p < FS * FN ? p / FN : FS;
}

struct Ring {
  unsigned char* base;  // 1024-aligned
  uint64_t* full;
  uint64_t* empty;
  int cs;        // next stage to consume (== next stage to fill between streams)
  unsigned cph;  // its fill parity
  int stride;    // bytes per stage (multiple of 1024)
  int nst;       // stages (<= MAX_STAGES)
  unsigned long long* dbg;  // optional: CTA 0 stream timeline accumulators (4 per stream slot)
  int dbg_slot;
};

__device__ __forceinline__ unsigned long long pr_clock() {
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
  r.cs = 0;
  r.cph = 0;
  r.stride = stride;
  r.nst = nst;
  r.dbg = nullptr;
  r.dbg_slot = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      tma::mbar_init(&r.full[s], 1);
      tma::mbar_init(&r.empty[s], blockDim.x / 32);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  return r;
}

// Operand boxes of a phase: box_a rows of A (from the region's first strip), box_b rows of B.
struct Boxes {
  const CUtensorMap* ma;
  const CUtensorMap* mb;
  int box_a, box_b;
};

// first A row of the region's box
__device__ __forceinline__ int arow_of(const Region& g) { return g.m0 + strip_of(g.pb, g.FM, g.FN) * 16; }

// Fill stage s (fill parity ph): wait until every consumer warp released the stage's previous
// fill (a fresh barrier passes the parity-1 wait at once), then issue the two boxes of k-tile
// number kt (counted in the region's rotated order).
__device__ __forceinline__ void issue(Ring& r, int s, unsigned ph, const Boxes& bx, const Region& g, int kt) {
  tma::mbar_wait(&r.empty[s], ph ^ 1u);
  unsigned char* st = r.base + (size_t)s * r.stride;
  tma::mbar_expect_tx(&r.full[s], (bx.box_a + bx.box_b) * 128);
  kt += g.rot;
  if (kt >= g.ke) kt -= g.ke - g.kb;
  tma::load_2d(st, bx.ma, kt * 16, arow_of(g), &r.full[s]);
  tma::load_2d(st + bx.box_a * 128, bx.mb, kt * 16, g.n0, &r.full[s]);
}

// 8-byte shared load when pred != 0, else the fallback value (one predicated LDS, no branch)
__device__ __forceinline__ double lds64_if(unsigned pred, unsigned addr, double fallback) {
  double v;
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n mov.f64 %0, %3;\n @p ld.shared.f64 %0, [%1];\n}\n"
      : "=d"(v)
      : "r"(addr), "r"(pred), "d"(fallback));
  return v;
}

// This warp's run of NP pairs inside a region (offsets in doubles inside the stage's A / B box,
// lane row included).  Pairs past the region are dropped at the store; they compute on the
// region's first pair (valid shared memory).
template <int NP>
struct Frags {
  int a0;          // DEDUPE: A offset of the first strip of the run
  int t1;          // DEDUPE: pairs of the run in its first strip (NP: the run stays in one strip)
  unsigned h1, h2; // DEDUPE: first / second strip of the run is the single-row last strip
  unsigned v0, v1; // bit j: first / second fragment of pair j inside the region
  unsigned hmask;  // bit j: pair j is horizontal (same A row, B columns c and c + 1)
  int aoff[NP];    // A offset of pair j's first fragment
  int boff[NP];    // B offset of pair j's first fragment
};

template <int NP>
__device__ __forceinline__ void frags_for(const Region& g, Frags<NP>& fr) {
  const int FS = g.FM >> 1, full = FS * g.FN;
  const int sf = strip_of(g.pb, g.FM, g.FN);
  const int warp = threadIdx.x >> 5, lr = (threadIdx.x & 31) >> 2;
  const int p0 = g.pb + warp * NP;
  fr.v0 = fr.v1 = fr.hmask = 0u;
  fr.h1 = fr.h2 = 0u;
  fr.t1 = NP;
  fr.a0 = lr * 16;
  int s_run = 0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const int p = p0 + j;
    const bool ok = p < g.pe;
    const int pp = ok ? p : g.pb;
    int s, c0;
    bool h;
    if (pp < full) {
      s = pp / g.FN;
      c0 = pp - s * g.FN;
      h = false;
    } else {
      s = FS;
      c0 = 2 * (pp - full);
      h = true;
    }
    if (j == 0) {
      s_run = s;
      fr.a0 = ((s - sf) * 16 + lr) * 16;
      fr.h1 = h ? 1u : 0u;
    } else if (ok && s != s_run && fr.t1 == NP) {
      fr.t1 = j;
      fr.h2 = h ? 1u : 0u;
    }
    fr.aoff[j] = ((s - sf) * 16 + lr) * 16;
    fr.boff[j] = (c0 * 8 + lr) * 16;
    if (h) fr.hmask |= 1u << j;
    if (ok) {
      fr.v0 |= 1u << j;
      if (!h || c0 + 1 < g.FN) fr.v1 |= 1u << j;
    }
  }
}

template <int NP, bool DEDUPE>
__device__ __forceinline__ void compute(const Ring& r, int s, const Boxes& bx, const Frags<NP>& fr,
                                        double (&acc)[2 * NP][2]) {
  const unsigned sA = tma::smem_u32(r.base) + s * r.stride;
  const unsigned sB = sA + bx.box_a * 128;
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const unsigned hv = fr.hmask & fr.v1;  // pairs whose second fragment needs its own B column
#pragma unroll
  for (int ks = 0; ks < 16; ks += 4) {
    const int off = tma::swz_off(ks >> 2, lr, lc);
    if constexpr (DEDUPE) {
      const unsigned pa = sA + (fr.a0 + off) * 8;
      const double x0 = tma::lds64(pa);
      const double x1 = lds64_if(fr.h1 ^ 1u, pa + 128 * 8, x0);
      const unsigned two = fr.t1 < NP ? 1u : 0u;
      const double x2 = lds64_if(two, pa + 256 * 8, x0);
      const double x3 = lds64_if(two & (fr.h2 ^ 1u), pa + 384 * 8, two ? x2 : x1);
      double b0[NP], b1[NP];
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const unsigned pb = sB + (fr.boff[j] + off) * 8;
        b0[j] = tma::lds64(pb);
        b1[j] = lds64_if((hv >> j) & 1u, pb + 128 * 8, b0[j]);
      }
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        tile::dmma(acc[2 * j], j < fr.t1 ? x0 : x2, b0[j]);
        tile::dmma(acc[2 * j + 1], j < fr.t1 ? x1 : x3, b1[j]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const unsigned pa = sA + (fr.aoff[j] + off) * 8, pb = sB + (fr.boff[j] + off) * 8;
        const unsigned h = (fr.hmask >> j) & 1u;
        const double a0 = tma::lds64(pa);
        const double b0 = tma::lds64(pb);
        // the pair's third operand: the next A row (vertical) or the next B column (horizontal)
        const double t = lds64_if(h ? (hv >> j) & 1u : 1u, h ? pb + 128 * 8 : pa + 128 * 8, b0);
        tile::dmma(acc[2 * j], a0, b0);
        tile::dmma(acc[2 * j + 1], h ? a0 : t, h ? t : b0);
      }
    }
  }
}

// Stream regions get(0..n-1) through the ring; epi(region, frags, acc) after each non-empty
// region's last k-tile (all threads call it).  Empty regions (pb >= pe) are skipped.
template <int NP, bool DEDUPE, class Get, class Epi>
__device__ __forceinline__ void stream(Ring& r, const Boxes& bx, int n, Get get, Epi epi) {
  const int lane = threadIdx.x & 31;
  const bool tl = r.dbg != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  const unsigned long long t_start = tl ? pr_clock() : 0;
  // producer cursor (thread 0): region, k-tile, stage and fill parity
  int pi = -1, pk = 0;
  Region P;
  P.kb = P.ke = 0;
  int ps = r.cs;
  unsigned pph = r.cph;
  const int nst = r.nst;
  auto p_next = [&]() {  // advance to the next non-empty region; false at the end
    while (++pi < n) {
      P = get(pi);
      if (P.pb < P.pe && P.kb < P.ke) {
        pk = P.kb;
        return true;
      }
    }
    return false;
  };
  bool p_live = false;
  auto produce = [&]() {
    issue(r, ps, pph, bx, P, pk);
    if (++ps == nst) {
      ps = 0;
      pph ^= 1u;
    }
    if (++pk >= P.ke) p_live = p_next();
  };
  if (threadIdx.x == 0) {
    tma::fence_proxy_async();  // earlier generic-proxy use of the ring's shared memory
    p_live = p_next();
    for (int s = 0; s < nst - 1 && p_live; ++s) produce();
  }
  __syncwarp();
  int cs = r.cs;
  unsigned cph = r.cph;
  bool first = true;
  for (int ci = 0; ci < n; ++ci) {
    const Region Cur = get(ci);
    if (!(Cur.pb < Cur.pe && Cur.kb < Cur.ke)) continue;
    Frags<NP> fr;
    frags_for<NP>(Cur, fr);
    double acc[2 * NP][2];
#pragma unroll
    for (int f = 0; f < 2 * NP; ++f) acc[f][0] = acc[f][1] = 0.0;
    for (int ck = Cur.kb; ck < Cur.ke; ++ck) {
      if (threadIdx.x == 0 && p_live) produce();
      __syncwarp();
      tma::mbar_wait(&r.full[cs], cph);
      if (tl && first) r.dbg[4 * r.dbg_slot] += pr_clock() - t_start;
      first = false;
      compute<NP, DEDUPE>(r, cs, bx, fr, acc);
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&r.empty[cs]);
      if (++cs == nst) {
        cs = 0;
        cph ^= 1u;
      }
    }
    if (tl) r.dbg[4 * r.dbg_slot + 1] += pr_clock() - t_start;
    epi(Cur, fr, acc);
    if (tl) r.dbg[4 * r.dbg_slot + 2] += pr_clock() - t_start;
  }
  __syncthreads();
  if (tl) r.dbg[4 * r.dbg_slot + 3] += pr_clock() - t_start;
  r.cs = cs;
  r.cph = cph;
}

// Store this warp's fragments of region g (limits M, N): rowptr(row) -> column 0 of row.
template <int NP, class RowPtr>
__device__ __forceinline__ void store(const Region& g, const Frags<NP>& fr, const double (&acc)[2 * NP][2], int M,
                                     int N, RowPtr&& rowptr) {
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
  const int arow0 = arow_of(g);
  const int clim = min(N, g.n0 + g.FN * 8);
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const bool h = (fr.hmask >> j) & 1u;
    const int row = arow0 + fr.aoff[j] / 16;
    const int col = g.n0 + (fr.boff[j] / 16 - lr) + lc * 2;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const bool ok = ((t == 0 ? fr.v0 : fr.v1) >> j) & 1u;
      const int rw = row + ((t == 1 && !h) ? 8 : 0);
      const int cl = col + ((t == 1 && h) ? 8 : 0);
      if (ok && rw < M) {
        double* dst = rowptr(rw);
        if (cl + 1 < clim) {
          dst[cl] = acc[2 * j + t][0];
          dst[cl + 1] = acc[2 * j + t][1];
        } else if (cl < clim) {
          dst[cl] = acc[2 * j + t][0];
        }
      }
    }
  }
}

// Pairs per warp for a region of P pairs.
__host__ __device__ inline int np_for(int P) { return (P + NWARP - 1) / NWARP; }
// A warp run of np pairs over strips of fn pairs spans at most 2 strips.
__host__ __device__ inline bool dedupe_ok(int np, int fn) { return np <= fn; }

}  // namespace tmapr
}  // namespace qtt
