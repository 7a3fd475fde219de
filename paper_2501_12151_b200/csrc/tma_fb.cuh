// Fragment-balanced TMA/DMMA engine for one-wave GEMM phases of a persistent kernel.
//
// The small local-system GEMMs of the AMEn sweep (e.g. 10400 x 100 x 200 at rank
// 100) are too small for fixed CTA tiles: rounding the tile count to the 148 SMs,
// and the warp count of a tile to the 4 schedulers per SM, idles up to half of the
// DMMA pipes (tools/tile_bench.cu).  Here each CTA gets an output REGION sized to
// its exact share of the work -- a run of 8x8 DMMA fragments of the row-major fragment
// grid (Region::fb, fe), or whole fragment rows / a column block -- and inside the
// region the fragments are dealt out to the 12 warps (3 per scheduler) in equal
// contiguous runs, so every scheduler issues the same number of DMMAs.  A warp keeps
// up to MAXF fragment accumulators; when its run spans at most 2 fragment rows the A
// fragments are loaded once per row and picked with a select.
//
// Operands are K-contiguous (C = A . B^T); per k-tile one TMA box of A rows and one
// of B rows (16 doubles of K each, 128B swizzle) land in a ring of run-time depth
// guarded by full/empty mbarriers.  The consumer loop is software-pipelined (the
// operands of the next k-step, also across a k-tile boundary, are loaded while the
// current k-step's DMMAs issue) and the TMA issue rotates over the warps (stream()).
#pragma once
#include "tma_tile.cuh"

// tools/tile_bench.cu builds the engine with -DQTT_FB_NOLOAD (no TMA copies: stale operands) and
// -DQTT_FB_NOSYNC (no mbarrier traffic at all) to separate the cost of the data supply and of the
// ring handshake from the consumer instruction stream itself.
#ifdef QTT_FB_NOSYNC
#define QTT_FB_WAIT(bar, parity) ((void)0)
#define QTT_FB_ARRIVE(bar) ((void)0)
#else
#define QTT_FB_WAIT(bar, parity) tma::mbar_wait(bar, parity)
#define QTT_FB_ARRIVE(bar) tma::mbar_arrive(bar)
#endif

namespace qtt {
namespace tmafb {

constexpr int MAXF = 16;   // fragments per warp (largest instantiation)
constexpr int NWARP = 12;  // consumer warps per CTA: 3 per scheduler (16 warps at 128 registers: no faster)
constexpr int MAX_STAGES = 8;  // deepest ring (run-time depth Ring::nst; look-ahead nst - 2 k-tiles)
constexpr int HEADER = 256;    // mbarriers (full + empty per stage) before the ring

// One unit of work: fragments [fb, fe) (row-major numbering) of the fragment grid covering
// output rows [m0, m0+mrows) x cols [n0, n0+ncols), over k-tiles [kb, ke).  fe = 0: the whole grid.
struct Region {
  int m0, mrows, n0, ncols, kb, ke, fb, fe;
};

struct Ring {
  unsigned char* base;  // 1024-aligned
  uint64_t* full;
  uint64_t* empty;
  int cs;                     // next stage to consume
  unsigned cph;               // its fill parity
  int stride;                 // bytes per stage (multiple of 1024)
  int nst;                    // stages (3 .. MAX_STAGES)
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
  r.cs = 0;
  r.cph = 0;
  r.stride = stride;
  r.nst = nst;
  r.dbg = nullptr;
  r.dbg_slot = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      tma::mbar_init(&r.full[s], 1);
      tma::mbar_init(&r.empty[s], NWARP);
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

// Fill stage s (fill parity ph) with k-tile kt of region g: wait until every consumer warp
// released the stage's previous fill (a fresh barrier passes the parity-1 wait at once).
__device__ __forceinline__ void issue(Ring& r, int s, unsigned ph, const Boxes& bx, const Region& g, int kt) {
  QTT_FB_WAIT(&r.empty[s], ph ^ 1u);
  unsigned char* st = r.base + (size_t)s * r.stride;
#ifdef QTT_FB_NOLOAD  // tools/tile_bench.cu: the loop without the TMA copies (stale operands)
  QTT_FB_ARRIVE(&r.full[s]);
  (void)st;
#else
  tma::mbar_expect_tx(&r.full[s], (bx.box_a + bx.box_b) * 128);
  tma::load_2d(st, bx.ma, kt * 16, g.m0, &r.full[s]);
  tma::load_2d(st + bx.box_a * 128, bx.mb, kt * 16, g.n0, &r.full[s]);
#endif
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
  int boff[NF];    // B fragment row offset in the stage (BYTES, incl. lane row)
  int aoff[NF];    // A fragment row offset (BYTES, incl. lane row)
  int ko[4];       // byte offset of this lane's 8-byte element in k-step 0..3 (128B swizzle)
};

template <int NF>
__device__ __forceinline__ void frags_for(const Region& g, Frags<NF>& fr) {
  const int FN = (g.ncols + 7) >> 3, FM = (g.mrows + 7) >> 3;
  const int F = g.fe > 0 ? g.fe : FM * FN;
  const int warp = threadIdx.x >> 5, lr = (threadIdx.x & 31) >> 2;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) fr.ko[ks] = tma::swz_off(ks, lr, threadIdx.x & 3) * 8;
  const int g0 = g.fb + warp * NF;
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
    fr.aoff[f] = (ii * 8 + lr) * 128;
    fr.boff[f] = (jj * 8 + lr) * 128;
    if (++j == FN) {
      j = 0;
      ++i;
    }
  }
}

// Operand fragments of one k-step, held in registers.
template <int NF, bool DEDUPE>
struct Operands {
  double b[NF];
  double a[2];  // DEDUPE: the run's two A fragment rows; else fragment 0's A (the rest follow one ahead)
};

// Load the operands of k-step ks (0..3) of the k-tile in stage s.
template <int NF, bool DEDUPE>
__device__ __forceinline__ void load_step(const Ring& r, int s, int ks, const Boxes& bx, const Frags<NF>& fr,
                                          Operands<NF, DEDUPE>& o) {
  const unsigned sA = tma::smem_u32(r.base) + s * r.stride + fr.ko[ks];
  const unsigned sB = sA + bx.box_a * 128;
  if constexpr (DEDUPE) {
    o.a[0] = tma::lds64(sA + fr.aoff[0]);
    o.a[1] = tma::lds64(sA + fr.aoff[0] + 1024);
  } else {
    o.a[0] = tma::lds64(sA + fr.aoff[0]);
  }
#pragma unroll
  for (int f = 0; f < NF; ++f) o.b[f] = tma::lds64(sB + fr.boff[f]);
}

// Issue the DMMAs of the k-step held in o and, when NEXT, replace every operand by that of
// k-step ks_n of stage s_n right after its last use: the loads of the next k-step (and of the next
// k-tile, whose full barrier the caller has already passed) are in flight while this step's
// DMMAs drain, so the warps never stand at a k-tile boundary with an empty DMMA queue (measured
// ~250 clocks per k-tile before, tools/micro/tma_rate.cu).
template <int NF, bool DEDUPE, bool NEXT>
__device__ __forceinline__ void step(const Ring& r, int s_c, int ks_c, int s_n, int ks_n, const Boxes& bx,
                                     const Frags<NF>& fr, Operands<NF, DEDUPE>& o, double (&acc)[NF][2]) {
  const unsigned sA = tma::smem_u32(r.base) + s_n * r.stride + fr.ko[ks_n];
  const unsigned sB = sA + bx.box_a * 128;
  if constexpr (DEDUPE) {
    double n0 = 0.0, n1 = 0.0;
    if constexpr (NEXT) {
      n0 = tma::lds64(sA + fr.aoff[0]);
      n1 = tma::lds64(sA + fr.aoff[0] + 1024);
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      tile::dmma(acc[f], f < fr.t1 ? o.a[0] : o.a[1], o.b[f]);
      if constexpr (NEXT) o.b[f] = tma::lds64(sB + fr.boff[f]);
    }
    if constexpr (NEXT) {
      o.a[0] = n0;
      o.a[1] = n1;
    }
  } else {
    // A fragments one ahead of their DMMA (this step's from the current stage s_c)
    const unsigned sAc = tma::smem_u32(r.base) + s_c * r.stride + fr.ko[ks_c];
    double a = o.a[0];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      double an = 0.0;
      if (f + 1 < NF)
        an = tma::lds64(sAc + fr.aoff[f + 1]);
      else if constexpr (NEXT)
        an = tma::lds64(sA + fr.aoff[0]);
      tile::dmma(acc[f], a, o.b[f]);
      if constexpr (NEXT) o.b[f] = tma::lds64(sB + fr.boff[f]);
      a = an;
    }
    o.a[0] = a;
  }
}

// Stream regions get(0..n-1) through the ring; epi(region, frags, acc) after each region's last
// k-tile (all threads call it).  The ring runs LA = nst - 2 k-tiles ahead and k-tile q is issued
// by lane 0 of warp q % NWARP at the top of k-tile q - LA: the stage it refills was released two
// k-tiles ago, so the issuing warp does not wait for the slowest warp, and the issue cost is paid
// by a different warp every k-tile.  (With thread 0 producing for everybody at a look-ahead of
// nst - 1, warp 0 waited for the slowest warp and issued on every k-tile, and every k-tile ran
// ~630 clocks behind its DMMA time -- profiles/r02/micro.)
template <int NF, bool DEDUPE, class Get, class Epi>
__device__ __forceinline__ void stream(Ring& r, const Boxes& bx, int n, Get get, Epi epi) {
  if (n <= 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool tl = r.dbg != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
  const unsigned long long t_start = tl ? fb_clock() : 0;
  const int nst = r.nst, LA = nst - 2;
  // producer cursor (tracked by every thread): region pi, k-tile pk, stage ps, fill parity pph,
  // issuing warp pw
  int pi = 0, ps = r.cs, pw = 0;
  unsigned pph = r.cph;
  Region P = get(0);
  int pk = P.kb;
  auto produce = [&]() {
    if (pi < n) {
      if (warp == pw && lane == 0) issue(r, ps, pph, bx, P, pk);
      if (++pk >= P.ke && ++pi < n) {
        P = get(pi);
        pk = P.kb;
      }
    }
    if (++ps == nst) {
      ps = 0;
      pph ^= 1u;
    }
    if (++pw == NWARP) pw = 0;
  };
  if (lane == 0) tma::fence_proxy_async();  // earlier generic-proxy use of the ring's shared memory
  for (int j = 0; j < LA; ++j) produce();
  __syncwarp();
  int cs = r.cs;
  unsigned cph = r.cph;
  for (int ci = 0; ci < n; ++ci) {
    const Region Cur = get(ci);
    Frags<NF> fr;
    frags_for<NF>(Cur, fr);
    double acc[NF][2];
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[f][0] = acc[f][1] = 0.0;
    Operands<NF, DEDUPE> o;
    // region prologue: the operands of its first k-step
    QTT_FB_WAIT(&r.full[cs], cph);
    if (tl && ci == 0) r.dbg[4 * r.dbg_slot] += fb_clock() - t_start;
    load_step<NF, DEDUPE>(r, cs, 0, bx, fr, o);
    for (int ck = Cur.kb; ck + 1 < Cur.ke; ++ck) {
      produce();
      __syncwarp();
      step<NF, DEDUPE, true>(r, cs, 0, cs, 1, bx, fr, o, acc);
      step<NF, DEDUPE, true>(r, cs, 1, cs, 2, bx, fr, o, acc);
      step<NF, DEDUPE, true>(r, cs, 2, cs, 3, bx, fr, o, acc);
      int ns = cs + 1;
      if (ns == nst) {
        ns = 0;
        cph ^= 1u;
      }
      // the last k-step loads from the next k-tile: pass its full barrier now (probing it three
      // k-steps earlier and waiting only on a failed probe measured the same)
      QTT_FB_WAIT(&r.full[ns], cph);
      step<NF, DEDUPE, true>(r, cs, 3, ns, 0, bx, fr, o, acc);
      __syncwarp();
      if (lane == 0) QTT_FB_ARRIVE(&r.empty[cs]);
      cs = ns;
    }
    {  // the region's last k-tile
      produce();
      __syncwarp();
      step<NF, DEDUPE, true>(r, cs, 0, cs, 1, bx, fr, o, acc);
      step<NF, DEDUPE, true>(r, cs, 1, cs, 2, bx, fr, o, acc);
      step<NF, DEDUPE, true>(r, cs, 2, cs, 3, bx, fr, o, acc);
      step<NF, DEDUPE, false>(r, cs, 3, cs, 0, bx, fr, o, acc);
      __syncwarp();
      if (lane == 0) QTT_FB_ARRIVE(&r.empty[cs]);
      if (++cs == nst) {
        cs = 0;
        cph ^= 1u;
      }
    }
    if (tl) r.dbg[4 * r.dbg_slot + 1] += fb_clock() - t_start;
    epi(Cur, fr, acc);
    if (tl) r.dbg[4 * r.dbg_slot + 2] += fb_clock() - t_start;
  }
  __syncthreads();
  if (tl) r.dbg[4 * r.dbg_slot + 3] += fb_clock() - t_start;
  r.cs = cs;
  r.cph = cph;
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
      const int row = g.m0 + fr.aoff[f] / 128;
      const int col = g.n0 + (fr.boff[f] / 128 - lr) + lc * 2;
      if (row < rlim) {
        double* dst = rowptr(row);
        if (col + 1 < clim) {
          if ((reinterpret_cast<uintptr_t>(dst + col) & 15) == 0) {
            *reinterpret_cast<double2*>(dst + col) = make_double2(acc[f][0], acc[f][1]);
          } else {
            dst[col] = acc[f][0];
            dst[col + 1] = acc[f][1];
          }
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
  return per <= 1 ? 1 : per <= 8 ? per : per <= 10 ? 10 : per <= 12 ? 12 : 16;
}
// A warp run of nf fragments over rows of fn fragments spans at most 2 rows.
__host__ __device__ inline bool dedupe_ok(int nf, int fn) { return nf <= fn + 1; }

}  // namespace tmafb
}  // namespace qtt
