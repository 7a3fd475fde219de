// Microbenchmark of the DMMA GEMM on the contraction-chain shapes of the sweep.
// Build: make -C paper_2501_12151_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -std=c++17 -I paper_2501_12151_b200/csrc tools/gemm_shapes.cu paper_2501_12151_b200/csrc/build/gemm.o
//   paper_2501_12151_b200/csrc/build/capi.o ... (see tools/build_tools.sh)
#include <cstdio>
#include <vector>

#include "contract.cuh"
#include "engine.cuh"
#include "gemm.cuh"

using namespace qtt;

static void fill_rand(double* d, long long n) {
  std::vector<double> h(n);
  unsigned s = 12345;
  for (auto& v : h) { s = s * 1103515245u + 12345u; v = ((s >> 8) & 0xffff) / 65536.0 - 0.5; }
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
}

int main() {
  Ctx c(0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct S { int r, R, n; };
  for (S sh : {S{32, 16, 2}, S{64, 16, 2}, S{128, 16, 2}, S{256, 16, 2}, S{36, 46, 2}, S{68, 49, 2},
               S{100, 52, 2}, S{196, 52, 2}}) {
    const int r = sh.r, R = sh.R, n = sh.n, m = n;
    DBuf phil((long long)r * R * r, c.stream), phir((long long)r * R * r, c.stream);
    DBuf A((long long)R * m * n * R, c.stream), Ap((long long)R * m * n * R, c.stream);
    DBuf x((long long)r * n * r, c.stream), y((long long)r * m * r, c.stream);
    fill_rand(phil.p, phil.n); fill_rand(phir.p, phir.n); fill_rand(A.p, A.n); fill_rand(x.p, x.n);
    permute_op_core(A.p, R, m, n, R, Ap.p, nullptr, c.stream);
    long long need = local_matvec_scratch(r, R, r, m, n, R, r, r) + (long long)r * m * r * 64;
    DBuf sc(need, c.stream);
    for (int w = 0; w < 3; ++w)
      local_matvec(phil.p, r, R, r, Ap.p, m, n, R, phir.p, r, r, x.p, y.p, 1.0, 0.0, {sc.p, sc.n}, c.stream);
    const int iters = 50;
    cudaEventRecord(e0, c.stream);
    for (int it = 0; it < iters; ++it)
      local_matvec(phil.p, r, R, r, Ap.p, m, n, R, phir.p, r, r, x.p, y.p, 1.0, 0.0, {sc.p, sc.n}, c.stream);
    cudaEventRecord(e1, c.stream);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = local_matvec_flops(r, R, r, m, n, R, r, r);
    // individual steps
    double* t1 = sc.p;
    double* t2 = sc.p + (long long)r * R * n * r;
    double* ws = t2 + (long long)r * m * R * r;
    long long wsn = sc.n - (ws - sc.p);
    GemmArgs g1; g1.M = r * R; g1.N = n * r; g1.K = r;
    gemm_set_A(g1, phil.p, r, false); gemm_set_B(g1, x.p, (long long)n * r, false); gemm_set_C(g1, t1, (long long)n * r);
    GemmArgs g2; g2.M = m * R; g2.N = r; g2.K = R * n;
    gemm_set_A(g2, Ap.p, (long long)R * n, false); gemm_set_B(g2, t1, r, false); g2.b_bs1 = (long long)R * n * r;
    gemm_set_C(g2, t2, r); g2.c_bs1 = (long long)m * R * r; g2.batch1 = r;
    GemmArgs g3; g3.M = r * m; g3.N = r; g3.K = R * r;
    gemm_set_A(g3, t2, (long long)R * r, false); gemm_set_B(g3, phir.p, (long long)R * r, true); gemm_set_C(g3, y.p, r);
    float mss[3];
    GemmArgs* gs[3] = {&g1, &g2, &g3};
    for (int s = 0; s < 3; ++s) {
      for (int w = 0; w < 3; ++w) gemm(*gs[s], c.stream, ws, wsn);
      cudaEventRecord(e0, c.stream);
      for (int it = 0; it < iters; ++it) gemm(*gs[s], c.stream, ws, wsn);
      cudaEventRecord(e1, c.stream);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&mss[s], e0, e1);
    }
    const double f1 = 2.0 * r * R * r * n * r, f2 = 2.0 * r * m * R * R * n * r, f3 = 2.0 * r * m * r * R * r;
    printf("{\"r\":%d,\"R\":%d,\"k1_us\":%.1f,\"k1_tflops\":%.2f,\"s1_us\":%.1f,\"s1_tf\":%.2f,\"s2_us\":%.1f,"
           "\"s2_tf\":%.2f,\"s3_us\":%.1f,\"s3_tf\":%.2f}\n",
           r, R, ms * 1000 / iters, fl / (ms / iters) / 1e9, mss[0] * 1000 / iters, f1 / (mss[0] / iters) / 1e9,
           mss[1] * 1000 / iters, f2 / (mss[1] / iters) / 1e9, mss[2] * 1000 / iters, f3 / (mss[2] / iters) / 1e9);
  }
  // a big square GEMM for reference
  for (int N : {2048, 4096}) {
    DBuf a((long long)N * N, c.stream), b((long long)N * N, c.stream), d((long long)N * N, c.stream);
    fill_rand(a.p, a.n); fill_rand(b.p, b.n);
    GemmArgs g; g.M = N; g.N = N; g.K = N;
    gemm_set_A(g, a.p, N, false); gemm_set_B(g, b.p, N, false); gemm_set_C(g, d.p, N);
    for (int w = 0; w < 2; ++w) gemm(g, c.stream);
    cudaEventRecord(e0, c.stream);
    for (int it = 0; it < 5; ++it) gemm(g, c.stream);
    cudaEventRecord(e1, c.stream);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"square\":%d,\"tflops\":%.2f}\n", N, 2.0 * N * N * (double)N / (ms / 5) / 1e9);
  }
  return 0;
}
