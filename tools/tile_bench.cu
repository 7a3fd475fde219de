// Throughput of the DMMA tile engine (dmma_tile.cuh) in isolation: G CTAs each
// stream `items` output tiles of a K-deep product from L2-resident operands.
// Reports per-k-tile time and DMMA-pipe fraction for 1 and 2 CTAs per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2501_12151_b200/csrc
//        tools/tile_bench.cu paper_2501_12151_b200/csrc/tma_map.cu -o tools/tile_bench
#include <cmath>
#include <cstdio>
#include <vector>

#include "dmma_tile.cuh"
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
  run_tma<tma::Cfg<64, 64, 2, 4, 3>>("64x64", M, N, K, A, B, C);
  run_tma<tma::Cfg<64, 64, 2, 4, 4>>("64x64s4", M, N, K, A, B, C);
  run_tma<tma::Cfg<64, 112, 4, 2, 3>>("64x112", M, N, K, A, B, C);
  run_tma<tma::Cfg<64, 112, 4, 2, 4>>("64x112s4", M, N, K, A, B, C);
  run_tma<tma::Cfg<128, 64, 4, 2, 3>>("128x64", M, N, K, A, B, C);
  run_tma<tma::Cfg<128, 112, 4, 2, 3>>("128x112", M, N, K, A, B, C);
  return 0;
}
