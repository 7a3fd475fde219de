// Throughput of the engine's DMMA GEMM (gemm.cu) on large and C4-chain shapes.
// Build: tools/build_tools.sh (links against the engine objects); run: tools/gemm_bench
#include <cstdio>
#include <vector>

#include "engine.cuh"
#include "gemm.cuh"

using namespace qtt;

int main() {
  Ctx c(0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct S { int M, N, K; const char* what; };
  for (S s : {S{4096, 4096, 4096, "square 4096"}, S{8192, 8192, 2048, "8192x8192x2048"},
              S{4096, 512, 256, "C4 r256 step1 (Phi_l . x)"}, S{512, 256, 4096, "C4 r256 step3 (t2 . Phi_r)"},
              S{2048, 256, 128, "C4 r128 step1"}, S{256, 128, 2048, "C4 r128 step3"},
              S{10406, 5000, 256, "QR outer update Y1-like"}}) {
    DBuf A((long long)s.M * s.K, c.stream), B((long long)s.K * s.N, c.stream), C((long long)s.M * s.N, c.stream);
    cudaMemsetAsync(A.p, 0, (size_t)s.M * s.K * 8, c.stream);
    cudaMemsetAsync(B.p, 0, (size_t)s.K * s.N * 8, c.stream);
    GemmArgs g;
    g.M = s.M; g.N = s.N; g.K = s.K;
    gemm_set_A(g, A.p, s.K, false);
    gemm_set_B(g, B.p, s.K, true);  // B stored [N][K]: K-contiguous operands (TMA-eligible)
    gemm_set_C(g, C.p, s.N);
    DBuf ws(gemm_workspace_hint(g) + 1, c.stream);
    for (int w = 0; w < 3; ++w) gemm(g, c.stream, ws.p, ws.n);
    cudaEventRecord(e0, c.stream);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) gemm(g, c.stream, ws.p, ws.n);
    cudaEventRecord(e1, c.stream);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double t = ms / 1e3 / reps;
    std::printf("%-28s M %5d N %5d K %5d: %8.1f us  %6.2f TFLOP/s\n", s.what, s.M, s.N, s.K, t * 1e6,
                2.0 * s.M * s.N * s.K / t / 1e12);
  }
  return 0;
}
