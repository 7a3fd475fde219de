// What limits the TMA -> mbarrier -> DMMA loop of the CG kernel?  148 CTAs x 384 threads stream KT
// k-tiles (one A box of ra rows + one B box of rb rows, 128 B per row) through an S-stage ring.
// Modes: compute NF fragments per warp per k-step (0 = just wait and release), B box shared by all
// CTAs or private, loads skipped entirely (barrier/loop overhead only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2501_12151_b200/csrc \
//   tools/micro/tma_rate.cu paper_2501_12151_b200/csrc/tma_map.cu -o tools/micro/tma_rate
#include <cstdio>
#include <cstdlib>

#include "tma_tile.cuh"

using namespace qtt;

struct Maps {
  alignas(64) CUtensorMap a;
  alignas(64) CUtensorMap b;
};

template <int NF>
__global__ void __launch_bounds__(384, 1) k(const __grid_constant__ Maps maps, int KT, int S, int ra, int rb,
                                            int stride, int shared_b, int noload, int iters, long long* clk,
                                            double* out) {
  extern __shared__ unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + 16;
  uintptr_t p = (reinterpret_cast<uintptr_t>(smem_raw) + 256 + 1023) & ~uintptr_t(1023);
  unsigned char* base = reinterpret_cast<unsigned char*>(p);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], 12);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lr = lane >> 2, lc = lane & 3;
  double acc[NF > 0 ? NF : 1][2];
  for (int f = 0; f < (NF > 0 ? NF : 1); ++f) acc[f][0] = acc[f][1] = 0.0;
  const int m0 = blockIdx.x * ra, n0 = shared_b ? 0 : blockIdx.x * rb;
  int ps = 0, cs = 0;
  unsigned pph = 0, cph = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    int pk = 0;
    auto produce = [&]() {
      tma::mbar_wait(&empty[ps], pph ^ 1u);
      unsigned char* st = base + (size_t)ps * stride;
      if (noload) {
        tma::mbar_arrive(&full[ps]);
      } else {
        tma::mbar_expect_tx(&full[ps], (ra + rb) * 128);
        tma::load_2d(st, &maps.a, pk * 16, m0, &full[ps]);
        tma::load_2d(st + ra * 128, &maps.b, pk * 16, n0, &full[ps]);
      }
      if (++ps == S) ps = 0, pph ^= 1u;
      ++pk;
    };
    if (threadIdx.x == 0)
      for (int s = 0; s < S - 1 && pk < KT; ++s) produce();
    __syncwarp();
    for (int kt = 0; kt < KT; ++kt) {
      if (threadIdx.x == 0 && pk < KT) produce();
      __syncwarp();
      tma::mbar_wait(&full[cs], cph);
      if constexpr (NF > 0) {
        const unsigned sA = tma::smem_u32(base) + cs * stride, sB = sA + ra * 128;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int off = tma::swz_off(ks, lr, lc);
          const double x0 = tma::lds64(sA + ((lr)*16 + off) * 8);
          double b[NF];
#pragma unroll
          for (int f = 0; f < NF; ++f) b[f] = tma::lds64(sB + ((((warp + f) % (rb / 8)) * 8 + lr) * 16 + off) * 8);
#pragma unroll
          for (int f = 0; f < NF; ++f) tile::dmma(acc[f], x0, b[f]);
        }
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[cs]);
      if (++cs == S) cs = 0, cph ^= 1u;
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  double s = 0;
  for (int f = 0; f < (NF > 0 ? NF : 1); ++f) s += acc[f][0] + acc[f][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int NF>
void run(int KT, int S, int ra, int rb, int shared_b, int noload, double* A, double* B, long long* clk, double* out,
         int ld = 0) {
  Maps maps;
  if (ld == 0) ld = KT * 16;
  make_tensor_map_2d(&maps.a, A, 148LL * ra, ld < KT * 16 ? ld : KT * 16, ld, ra);
  make_tensor_map_2d(&maps.b, B, shared_b ? rb : 148LL * rb, ld < KT * 16 ? ld : KT * 16, ld, rb);
  printf("ld %d: ", ld);
  const int stride = (((ra + rb) * 128 + 1023) / 1024) * 1024;
  const size_t smem = (size_t)S * stride + 256 + 1024;
  cudaFuncSetAttribute(k<NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 20;
  for (int rep = 0; rep < 2; ++rep) k<NF><<<148, 384, smem>>>(maps, KT, S, ra, rb, stride, shared_b, noload, iters, clk, out);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  const double per_pass = (double)h / iters, per_kt = per_pass / KT;
  printf("KT %3d S %2d ra %3d rb %3d sharedB %d noload %d NF %2d: %.0f clk/pass, %.0f clk/k-tile (DMMA issue %d), "
         "%.1f B/clk/SM %s\n", KT, S, ra, rb, shared_b, noload, NF, per_pass, per_kt, NF * 4 * 48,
         (ra + rb) * 128.0 / per_kt, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *A, *B, *out;
  long long* clk;
  cudaMalloc(&A, 148LL * 128 * 5200 * 8);
  cudaMalloc(&B, 148LL * 128 * 5200 * 8);
  cudaMemset(A, 0, 148LL * 128 * 5200 * 8);
  cudaMemset(B, 0, 148LL * 128 * 5200 * 8);
  cudaMalloc(&out, 1 << 22);
  cudaMalloc(&clk, 8);
  printf("-- row pitch 1600 B (rows alternate 0 / 64 B off a 128 B line) vs 1664 B\n");
  for (int ld : {200, 208}) {
    run<0>(13, 4, 72, 104, 1, 0, A, B, clk, out, ld);
    run<4>(13, 4, 8, 104, 1, 0, A, B, clk, out, ld);
    run<8>(13, 4, 48, 104, 1, 0, A, B, clk, out, ld);
    run<10>(13, 4, 72, 104, 1, 0, A, B, clk, out, ld);
  }
  for (int KT : {13}) {
    printf("-- pure streaming (no compute)\n");
    for (int S : {2, 4, 8}) {
      run<0>(KT, S, 72, 104, 1, 0, A, B, clk, out);
      run<0>(KT, S, 72, 104, 0, 0, A, B, clk, out);
      run<0>(KT, S, 8, 104, 1, 0, A, B, clk, out);
    }
    printf("-- loop/barrier overhead only (no loads)\n");
    run<0>(KT, 4, 72, 104, 1, 1, A, B, clk, out);
    run<4>(KT, 4, 72, 104, 1, 1, A, B, clk, out);
    run<10>(KT, 4, 72, 104, 1, 1, A, B, clk, out);
    printf("-- loads + compute\n");
    for (int S : {3, 4, 8}) {
      run<4>(KT, S, 8, 104, 1, 0, A, B, clk, out);
      run<4>(KT, S, 24, 104, 1, 0, A, B, clk, out);
      run<8>(KT, S, 48, 104, 1, 0, A, B, clk, out);
      run<10>(KT, S, 72, 104, 1, 0, A, B, clk, out);
      run<10>(KT, S, 72, 104, 0, 0, A, B, clk, out);
    }
  }
  return 0;
}
