// DMMA m8n8k4 issue/latency microbenchmark: one CTA of W warps, every warp runs ITERS rounds of
// NACC independent accumulator chains.  Prints clocks per round and per DMMA (SM-wide).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/dmma_lat tools/micro/dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void chain(double* out, long long* clk, int iters) {
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int NACC>
void run(int warps, double* out, long long* clk) {
  const int iters = 2000;
  chain<NACC><<<1, warps * 32>>>(out, clk, iters);
  chain<NACC><<<1, warps * 32>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  printf("warps %2d nacc %2d: %.1f clk/round, %.2f clk per DMMA SM-wide\n", warps, NACC, (double)h / iters,
         (double)h / iters / (NACC * warps));
}

int main() {
  double* out;
  long long* clk;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&clk, 8);
  for (int w : {1, 2, 4, 8, 12, 16}) {
    run<1>(w, out, clk);
    run<2>(w, out, clk);
    run<4>(w, out, clk);
    run<8>(w, out, clk);
    run<16>(w, out, clk);
  }
  return 0;
}
