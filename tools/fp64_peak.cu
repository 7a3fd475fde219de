// FP64 peak microbenchmark for B200 (sm_100a): DFMA pipe and DMMA (mma.sync f64) pipe.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// Prints one JSON line per measurement.  Used to fill the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
  for (int j = 0; j < 8; j++) a[j] = threadIdx.x * 1e-7 + j;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = fma(a[j], b, c);
  }
  double s = 0;
  for (int j = 0; j < 8; j++) s += a[j];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-7, b0 = 1e-3;
  double c[4][2];
  for (int j = 0; j < 4; j++) c[j][0] = c[j][1] = 0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a0), "d"(b0));
  }
  double s = 0;
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 1 << 20);
  int dev; cudaGetDevice(&dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps; int iters = 1 << 16;
      dfma_kernel<<<blocks, threads>>>(d, 16);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * (double)iters * blocks * threads;
      printf("{\"what\":\"dfma\",\"threads\":%d,\"blocks\":%d,\"tflops\":%.3f}\n", threads, blocks, flops / ms / 1e9);
      dmma_kernel<<<blocks, threads>>>(d, 16);
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(d, iters / 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 8 * 8 * 4 * 4 * (double)(iters / 4) * blocks * (threads / 32);
      printf("{\"what\":\"dmma_m8n8k4\",\"threads\":%d,\"blocks\":%d,\"tflops\":%.3f}\n", threads, blocks, flops / ms / 1e9);
    }
  }
  printf("{\"sms\":%d,\"clock_khz\":%d}\n", sms, p.clockRate);
  return 0;
}
