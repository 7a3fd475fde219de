// DMMA rate when operands come from shared memory: 12 warps, each k-step loads NB B fragments and
// NA A fragments (8-byte LDS, conflict-free swizzled pattern) and issues NF = NA * NB' DMMAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/dmma_lds tools/micro/dmma_lds.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int swz_off(int s, int lr, int lc) {
  const int chunk = (s + ((lc >> 1) << 2)) ^ lr;
  return (chunk << 1) | (lc & 1);
}

// MI x NI register block per warp: MI A loads + NI B loads, MI*NI DMMAs per k-step
template <int MI, int NI>
__global__ void __launch_bounds__(384, 1) blocked(double* out, long long* clk, int iters) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 24 * 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  double acc[MI][NI][2];
  for (int i = 0; i < MI; ++i) for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int aoff[MI], boff[NI];
  for (int i = 0; i < MI; ++i) aoff[i] = ((warp % 4 * MI + i) * 8 + lr) * 16;
  for (int j = 0; j < NI; ++j) boff[j] = 8192 + ((warp / 4 * NI + j) * 8 + lr) * 16;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const unsigned st = base + (it & 3) * 2048 * 8 * 0;  // same stage (no TMA here)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int off = swz_off(ks, lr, lc);
      double a[MI], b[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = lds64(st + (aoff[i] + off) * 8);
#pragma unroll
      for (int j = 0; j < NI; ++j) b[j] = lds64(st + (boff[j] + off) * 8);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < MI; ++i) for (int j = 0; j < NI; ++j) s += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int MI, int NI>
void run(double* out, long long* clk) {
  const int iters = 1000;
  cudaFuncSetAttribute(blocked<MI, NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int rep = 0; rep < 2; ++rep) blocked<MI, NI><<<148, 384, 200 * 1024>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / iters / 4;  // clocks per k-step
  printf("MI %d NI %d: loads %2d dmma %2d per k-step: %.1f clk/k-step, DMMA pipe %.0f%% (ideal %d clk) %s\n", MI, NI,
         MI + NI, MI * NI, per, 100.0 * MI * NI * 48 / per, MI * NI * 48, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out;
  long long* clk;
  cudaMalloc(&out, 1 << 22);
  cudaMalloc(&clk, 8);
  run<1, 4>(out, clk);
  run<1, 6>(out, clk);
  run<1, 8>(out, clk);
  run<1, 10>(out, clk);
  run<1, 16>(out, clk);
  run<2, 2>(out, clk);
  run<2, 3>(out, clk);
  run<2, 4>(out, clk);
  run<2, 5>(out, clk);
  run<2, 6>(out, clk);
  run<2, 8>(out, clk);
  run<4, 4>(out, clk);
  run<4, 2>(out, clk);
  run<3, 4>(out, clk);
  return 0;
}
