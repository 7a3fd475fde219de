// Throughput of the DMMA tile engine (dmma_tile.cuh) in isolation: G CTAs each
// stream `items` output tiles of a K-deep product from L2-resident operands.
// Reports per-k-tile time and DMMA-pipe fraction for 1 and 2 CTAs per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2501_12151_b200/csrc
//        tools/tile_bench.cu paper_2501_12151_b200/csrc/tma_map.cu -o tools/tile_bench
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include "dmma_tile.cuh"
#include "tma_fb.cuh"
#include "tma_rt.cuh"
#include "tma_tile.cuh"

using namespace qtt;

template <class T>
__global__ void __launch_bounds__(T::NT) bench_kernel(const double* A, const double* B, double* C, int M, int N,
                                                      int K, int items, bool a_kcontig) {
  extern __shared__ double smem[];
  tile::Operands o{A, a_kcontig ? (long long)K : 1, a_kcontig ? 1 : (long long)M, B, N, 1, M, N, K};
  const int tm = (M + T::BM - 1) / T::BM, tn = (N + T::BN - 1) / T::BN;
  const int ktiles = (K + T::BK - 1) / T::BK;
  auto get = [&](int i) {
    tile::TileItem t;
    t.o = o;
    const int it = (blockIdx.x + i * gridDim.x) % (tm * tn);
    t.m0 = (it / tn) * T::BM;
    t.n0 = (it % tn) * T::BN;
    t.kb = 0;
    t.ke = ktiles;
    return t;
  };
  auto epi = [&](const tile::TileItem& t, const double (&acc)[T::MI][T::NI][2]) {
    tile::for_each_acc<T>(t.m0, t.n0, M, N, acc, [&](int r, int c, double v) { C[(long long)r * N + c] = v; });
  };
  tile::mma_stream<T>(items, get, epi, smem);
}

template <class T>
void run(const char* name, int M, int N, int K, bool a_kcontig, double* A, double* B, double* C) {
  cudaFuncSetAttribute(bench_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ktiles = (K + T::BK - 1) / T::BK;
  for (int per_sm : {1, 2}) {
    for (int items : {1, 4}) {
      const int G = 148 * per_sm;
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        bench_kernel<T><<<G, T::NT, T::SMEM>>>(A, B, C, M, N, K, items, a_kcontig);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double flops = 2.0 * T::BM * T::BN * T::BK * ktiles * items * (double)G;
      printf("{\"tile\":\"%s\",\"a_kcontig\":%d,\"K\":%d,\"ctas_per_sm\":%d,\"items\":%d,\"us\":%.2f,"
             "\"us_per_ktile\":%.3f,\"tflops_padded\":%.2f,\"err\":\"%s\"}\n",
             name, a_kcontig ? 1 : 0, K, per_sm, items, best * 1e3, best * 1e3 / (ktiles * items),
             flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
}

struct TmaMaps {
  alignas(64) CUtensorMap a;
  alignas(64) CUtensorMap b;
};

template <class T>
__global__ void __launch_bounds__(T::NT) bench_tma_kernel(const __grid_constant__ TmaMaps maps, double* C, int M,
                                                          int N, int K, int items) {
  extern __shared__ unsigned char smem_raw[];
  tma::Ring ring = tma::ring_init<T::STAGES>(smem_raw);
  const int tm = (M + T::BM - 1) / T::BM, tn = (N + T::BN - 1) / T::BN;
  const int ktiles = (K + 15) / 16;
  auto get = [&](int i) {
    tma::Item t;
    t.ma = &maps.a;
    t.mb = &maps.b;
    const int it = (blockIdx.x + i * gridDim.x) % (tm * tn);
    t.m0 = (it / tn) * T::BM;
    t.n0 = (it % tn) * T::BN;
    t.kb = 0;
    t.ke = ktiles;
    return t;
  };
  auto epi = [&](const tma::Item& t, const double (&acc)[T::MI][T::NI][2]) {
    tma::for_each<T>(t.m0, t.n0, M, N, acc, [&](int r, int c, double v) { C[(long long)r * N + c] = v; });
  };
  tma::stream<T>(ring, items, get, epi);
}

template <class T>
void run_tma(const char* name, int M, int N, int K, double* A, double* B, double* C) {
  TmaMaps maps;
  make_tensor_map_2d(&maps.a, A, M, K, K, T::BM);
  make_tensor_map_2d(&maps.b, B, N, K, K, T::BN);
  cudaFuncSetAttribute(bench_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ktiles = (K + 15) / 16;
  for (int per_sm : {1, 2}) {
    for (int items : {1, 4}) {
      const int G = 148 * per_sm;
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        bench_tma_kernel<T><<<G, T::NT, T::SMEM>>>(maps, C, M, N, K, items);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double flops = 2.0 * T::BM * T::BN * 16 * ktiles * items * (double)G;
      printf("{\"tile\":\"tma%s\",\"K\":%d,\"ctas_per_sm\":%d,\"items\":%d,\"us\":%.2f,"
             "\"us_per_ktile\":%.3f,\"tflops_padded\":%.2f,\"err\":\"%s\"}\n",
             name, K, per_sm, items, best * 1e3, best * 1e3 / (ktiles * items), flops / (best * 1e-3) / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}

__global__ void __launch_bounds__(256, 1) bench_rt_kernel(const __grid_constant__ TmaMaps maps, double* C, int M,
                                                           int N, int K, int items, int wm, int wn, int stride) {
  extern __shared__ unsigned char smem_raw[];
  tmart::Ring ring = tmart::ring_init(smem_raw, stride);
  const tmart::Shape sh{wm, wn};
  const int BM = tmart::shape_bm(sh), BN = tmart::shape_bn(sh);
  const int tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  const int ktiles = (K + 15) / 16;
  const int total = tm * tn;
  const int mine = total * items > (int)blockIdx.x ? (total * items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto get = [&](int i) {
    tma::Item t;
    t.ma = &maps.a;
    t.mb = &maps.b;
    const int it = (blockIdx.x + i * gridDim.x) % total;
    t.m0 = (it / tn) * BM;
    t.n0 = (it % tn) * BN;
    t.kb = 0;
    t.ke = ktiles;
    return t;
  };
  auto epi = [&](const tma::Item& t, const double (&acc)[tmart::MI][tmart::NI][2]) {
    tmart::store_rows(sh, t.m0, t.n0, M, N, acc, [&](int r) { return C + (long long)r * N; });
  };
  tmart::stream(ring, sh, mine, get, epi);
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// fragment-balanced engine: every CTA streams `items` regions of rb x cb fragments
template <int NF, bool DD>
__global__ void __launch_bounds__(384, 1) bench_fb_kernel(const __grid_constant__ TmaMaps maps, double* C, int M,
                                                           int N, int K, int items, int rb, int cb, int stride) {
  extern __shared__ unsigned char smem_raw[];
  tmafb::Ring ring = tmafb::ring_init(smem_raw, stride, 6);
  const int FR = (M + 7) / 8, FC = (N + 7) / 8;
  const int nrb = (FR + rb - 1) / rb, ncb = (FC + cb - 1) / cb;
  const int KT = (K + 15) / 16;
  const tmafb::Boxes bx{&maps.a, &maps.b, rb * 8, cb * 8};
  auto get = [&](int i) {
    const int t = (blockIdx.x + i * gridDim.x) % (nrb * ncb);
    const int r = t / ncb, c = t % ncb;
    tmafb::Region g;
    g.m0 = r * rb * 8;
    g.mrows = min(rb, FR - r * rb) * 8;
    g.n0 = c * cb * 8;
    g.ncols = min(cb, FC - c * cb) * 8;
    g.kb = 0;
    g.ke = KT;
    g.fb = 0;
    g.fe = 0;
    return g;
  };
  auto epi = [&](const tmafb::Region& g, const auto& fr, const auto& acc) {
    tmafb::store(g, fr, acc, M, N, [&](int r) { return C + (long long)r * N; });
  };
  tmafb::stream<NF, DD>(ring, bx, items, get, epi);
}

template <int NF, bool DD>
void run_fb(int M, int N, int K, int rb, int cb, int items, double* A, double* B, double* C) {
  TmaMaps maps;
  make_tensor_map_2d(&maps.a, A, M, K, K, rb * 8);
  make_tensor_map_2d(&maps.b, B, N, K, K, cb * 8);
  const int stride = (((rb + cb) * 8 * 128 + 1023) / 1024) * 1024;
  const size_t smem = (size_t)6 * stride + tmafb::HEADER + 1024 + 4096;
  cudaFuncSetAttribute(bench_fb_kernel<NF, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 7; ++rep) {
    cudaEventRecord(e0);
    bench_fb_kernel<NF, DD><<<148, 384, smem>>>(maps, C, M, N, K, items, rb, cb, stride);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const int KT = (K + 15) / 16;
  // DMMA issue model: NF frags x 4 k-steps x KT x 3 warps per scheduler x 16 clk
  const double model_us = (double)NF * 4 * KT * 3 * 16 / 1965.0 * items;
  printf("{\"fb\":\"%dx%d\",\"nf\":%d,\"dedupe\":%d,\"K\":%d,\"items\":%d,\"us\":%.2f,\"model_us\":%.2f,"
         "\"err\":\"%s\"}\n", rb, cb, NF, DD ? 1 : 0, K, items, best * 1e3, model_us,
         cudaGetErrorString(cudaGetLastError()));
}

// CTA 0 timeline of one single-wave pass: timestamps after each full-barrier wait
__global__ void __launch_bounds__(256, 1) timeline_kernel(const __grid_constant__ TmaMaps maps, int K, int wm, int wn,
                                                           int stride, unsigned long long* ts) {
  extern __shared__ unsigned char smem_raw[];
  const unsigned long long t0 = gtime();
  tmart::Ring r = tmart::ring_init(smem_raw, stride);
  const tmart::Shape sh{wm, wn};
  const int KT = (K + 15) / 16;
  tma::Item it;
  it.ma = &maps.a;
  it.mb = &maps.b;
  it.m0 = blockIdx.x * tmart::shape_bm(sh);
  it.n0 = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool active = warp < wm * wn;
  const int wm0 = (warp % wm) * tmart::WROWS, wn0 = (warp / wm) * tmart::WCOLS;
  double acc[tmart::MI][tmart::NI][2];
  tmart::zero(acc);
  unsigned produced = 0;
  if (threadIdx.x == 0)
    for (int s = 0; s < 3 && (int)produced < KT; ++s) tmart::issue(r, produced, it, produced, sh), ++produced;
  __syncwarp();
  if (blockIdx.x == 0 && threadIdx.x == 0) ts[0] = gtime() - t0;
  for (int kt = 0; kt < KT; ++kt) {
    if (threadIdx.x == 0 && (int)produced < KT) tmart::issue(r, produced, it, produced, sh), ++produced;
    __syncwarp();
    tma::mbar_wait(&r.full[kt % 4], (kt / 4) & 1u);
    if (blockIdx.x == 0 && threadIdx.x == 0) ts[1 + kt] = gtime() - t0;
    if (active) tmart::compute(r, kt, acc, sh, wm0, wn0);
    __syncwarp();
    if (lane == 0) tma::mbar_arrive(&r.empty[kt % 4]);
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) ts[1 + KT] = gtime() - t0;
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < tmart::MI; ++i)
#pragma unroll
    for (int j = 0; j < tmart::NI; ++j) sum += acc[i][j][0] + acc[i][j][1];
  if (sum == 12345.0) ts[0] = 1;
}

void run_timeline(int M, int N, int K, int wm, int wn, double* A, double* B) {
  const tmart::Shape sh{wm, wn};
  TmaMaps maps;
  make_tensor_map_2d(&maps.a, A, M, K, K, tmart::shape_bm(sh));
  make_tensor_map_2d(&maps.b, B, N, K, K, tmart::shape_bn(sh));
  const int stride = ((tmart::stage_bytes(sh) + 1023) / 1024) * 1024;
  const size_t smem = (size_t)4 * stride + 64 + 1024;
  cudaFuncSetAttribute(timeline_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  const int KT = (K + 15) / 16;
  const int tiles = (M + tmart::shape_bm(sh) - 1) / tmart::shape_bm(sh);
  for (int rep = 0; rep < 3; ++rep) timeline_kernel<<<tiles, 256, smem>>>(maps, K, wm, wn, stride, d);
  cudaDeviceSynchronize();
  unsigned long long h[64];
  cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
  printf("{\"timeline\":\"%dx%d\",\"ns\":[", tmart::shape_bm(sh), tmart::shape_bn(sh));
  for (int i = 0; i <= KT + 1; ++i) printf("%s%llu", i ? "," : "", h[i]);
  printf("],\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
}

// one GEMM C[M][N] = A[M][K] . B[N][K]^T over all tiles (items = waves of tiles)
void run_rt(int M, int N, int K, int wm, int wn, int items, double* A, double* B, double* C) {
  const tmart::Shape sh{wm, wn};
  TmaMaps maps;
  make_tensor_map_2d(&maps.a, A, M, K, K, tmart::shape_bm(sh));
  make_tensor_map_2d(&maps.b, B, N, K, K, tmart::shape_bn(sh));
  const int stride = ((tmart::stage_bytes(sh) + 1023) / 1024) * 1024;
  const size_t smem = (size_t)4 * stride + 64 + 1024;
  cudaFuncSetAttribute(bench_rt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 7; ++rep) {
    cudaEventRecord(e0);
    bench_rt_kernel<<<148, 256, smem>>>(maps, C, M, N, K, items, wm, wn, stride);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const int tiles = ((M + tmart::shape_bm(sh) - 1) / tmart::shape_bm(sh)) * ((N + tmart::shape_bn(sh) - 1) / tmart::shape_bn(sh));
  const double flops = 2.0 * M * N * (double)K * items;
  printf("{\"rt\":\"%dx%d\",\"M\":%d,\"N\":%d,\"K\":%d,\"tiles\":%d,\"items\":%d,\"us\":%.2f,\"tflops_useful\":%.2f,"
         "\"err\":\"%s\"}\n", tmart::shape_bm(sh), tmart::shape_bn(sh), M, N, K, tiles, items, best * 1e3,
         flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

// correctness of the TMA engine against a host product on a small ragged case
int check_tma() {
  const int M = 150, N = 70, K = 53;
  std::vector<double> a((size_t)M * K), b((size_t)N * K), c((size_t)M * N);
  for (size_t i = 0; i < a.size(); ++i) a[i] = (double)((i * 37) % 101) / 101.0 - 0.5;
  for (size_t i = 0; i < b.size(); ++i) b[i] = (double)((i * 53) % 97) / 97.0 - 0.5;
  // K padded to an even stride for the 16-byte TMA stride rule
  const int ld = K + 1;
  std::vector<double> ap((size_t)M * ld, 0.0), bp((size_t)N * ld, 0.0);
  for (int i = 0; i < M; ++i) for (int k = 0; k < K; ++k) ap[(size_t)i * ld + k] = a[(size_t)i * K + k];
  for (int i = 0; i < N; ++i) for (int k = 0; k < K; ++k) bp[(size_t)i * ld + k] = b[(size_t)i * K + k];
  double *dA, *dB, *dC;
  cudaMalloc(&dA, ap.size() * 8);
  cudaMalloc(&dB, bp.size() * 8);
  cudaMalloc(&dC, c.size() * 8);
  cudaMemcpy(dA, ap.data(), ap.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, bp.data(), bp.size() * 8, cudaMemcpyHostToDevice);
  using T = tma::Cfg<64, 64, 2, 4, 3>;
  TmaMaps maps;
  make_tensor_map_2d(&maps.a, dA, M, K, ld, T::BM);
  make_tensor_map_2d(&maps.b, dB, N, K, ld, T::BN);
  cudaFuncSetAttribute(bench_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM);
  const int tiles = ((M + 63) / 64) * ((N + 63) / 64);
  bench_tma_kernel<T><<<tiles, T::NT, T::SMEM>>>(maps, dC, M, N, K, 1);
  cudaMemcpy(c.data(), dC, c.size() * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += a[(size_t)i * K + k] * b[(size_t)j * K + k];
      err = fmax(err, fabs(s - c[(size_t)i * N + j]));
    }
  printf("{\"tma_check_max_abs_err\":%.3e,\"err\":\"%s\"}\n", err, cudaGetErrorString(cudaGetLastError()));
  return err < 1e-12 ? 0 : 1;
}

int main() {
  if (getenv("TB_FB16")) {
    double *A, *B, *C;
    cudaMalloc(&A, (size_t)10400 * 1600 * 8);
    cudaMalloc(&B, (size_t)1600 * 256 * 8);
    cudaMalloc(&C, (size_t)10400 * 112 * 8);
    const int v = atoi(getenv("TB_FB16"));
    if (v == 1) run_fb<16, false>(10400, 100, 200, 9, 13, 1, A, B, C);
    if (v == 2) run_fb<16, true>(10400, 100, 200, 9, 13, 1, A, B, C);
    if (v == 3) run_fb<12, false>(10400, 100, 200, 9, 13, 1, A, B, C);
    if (v == 4) run_fb<16, false>(10400, 100, 200, 9, 16, 1, A, B, C);
    if (v == 5) run_fb<12, true>(10400, 100, 200, 9, 13, 1, A, B, C);
    if (v == 6) run_fb<10, true>(10400, 100, 200, 9, 13, 8, A, B, C);
    if (v == 7) run_fb<10, false>(10400, 100, 200, 9, 13, 8, A, B, C);
    if (v == 8) run_fb<10, true>(10400, 100, 1600, 9, 13, 1, A, B, C);
    if (v == 9) run_fb<8, true>(10400, 100, 1600, 8, 12, 1, A, B, C);
    if (v == 11) {
      run_fb<10, true>(10400, 100, 1600, 9, 13, 1, A, B, C);
      run_fb<10, false>(10400, 100, 1600, 9, 13, 1, A, B, C);
      run_fb<8, true>(10400, 100, 1600, 7, 13, 1, A, B, C);
      run_fb<8, false>(10400, 100, 1600, 7, 13, 1, A, B, C);
      run_fb<6, true>(10400, 100, 1600, 5, 13, 1, A, B, C);
      run_fb<6, false>(10400, 100, 1600, 5, 13, 1, A, B, C);
      run_fb<4, true>(10400, 100, 1600, 3, 13, 1, A, B, C);
      run_fb<4, false>(10400, 100, 1600, 3, 13, 1, A, B, C);
      run_fb<6, false>(1040, 200, 1600, 13, 5, 1, A, B, C);
      run_fb<8, false>(1040, 200, 1600, 13, 7, 1, A, B, C);
      run_fb<12, true>(10400, 100, 1600, 11, 13, 1, A, B, C);
      run_fb<16, false>(10400, 100, 1600, 14, 13, 1, A, B, C);
    }
    printf("v=%d %s\n", v, cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
  }
  if (check_tma()) return 1;
  const int M = 10400, N = 112, K = 208;
  double *A, *B, *C;
  cudaMalloc(&A, (size_t)M * K * 8);
  cudaMalloc(&B, (size_t)K * N * 8);
  cudaMalloc(&C, (size_t)M * N * 8);
  cudaMemset(A, 0, (size_t)M * K * 8);
  cudaMemset(B, 0, (size_t)K * N * 8);
  run<tile::Cfg<64, 64, 16, 2, 4, 3>>("64x64", M, N, K, true, A, B, C);
  run<tile::Cfg<64, 112, 16, 4, 2, 3>>("64x112", M, N, K, true, A, B, C);
  run<tile::Cfg<64, 112, 16, 4, 2, 4>>("64x112s4", M, N, K, true, A, B, C);
  run<tile::Cfg<128, 64, 16, 4, 2, 3>>("128x64", M, N, K, true, A, B, C);
  run<tile::Cfg<64, 64, 16, 2, 4, 3>>("64x64", M, N, K, false, A, B, C);
  run<tile::Cfg<64, 112, 16, 4, 2, 3>>("64x112", M, N, K, false, A, B, C);
  run<tile::Cfg<64, 64, 32, 2, 4, 3>>("64x64k32", M, N, K, true, A, B, C);
  for (int items : {1, 8}) {
    run_fb<10, true>(10400, 100, 200, 9, 13, items, A, B, C);
    run_fb<10, false>(10400, 100, 200, 9, 13, items, A, B, C);
    run_fb<16, false>(10400, 100, 200, 9, 13, items, A, B, C);
    run_fb<8, true>(10400, 100, 200, 8, 12, items, A, B, C);
    run_fb<4, true>(10400, 100, 200, 4, 12, items, A, B, C);
  }
  run_timeline(10400, 100, 200, 3, 2, A, B);
  run_timeline(10400, 100, 200, 5, 1, A, B);
  for (int items : {1, 4}) {
    run_rt(10400, 100, 200, 5, 1, items, A, B, C);
    run_rt(10400, 100, 200, 3, 2, items, A, B, C);
    run_rt(10400, 100, 200, 4, 2, items, A, B, C);
    run_rt(10400, 100, 200, 8, 1, items, A, B, C);
    run_rt(10400, 100, 200, 2, 2, items, A, B, C);
  }
  run_tma<tma::Cfg<64, 64, 2, 4, 3>>("64x64", M, N, K, A, B, C);
  run_tma<tma::Cfg<64, 64, 2, 4, 4>>("64x64s4", M, N, K, A, B, C);
  run_tma<tma::Cfg<64, 112, 4, 2, 3>>("64x112", M, N, K, A, B, C);
  run_tma<tma::Cfg<64, 112, 4, 2, 4>>("64x112s4", M, N, K, A, B, C);
  run_tma<tma::Cfg<128, 64, 4, 2, 3>>("128x64", M, N, K, A, B, C);
  run_tma<tma::Cfg<128, 112, 4, 2, 3>>("128x112", M, N, K, A, B, C);
  return 0;
}
