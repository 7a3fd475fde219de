// Cost of a grid-wide barrier on B200: cooperative_groups grid.sync() vs a
// generation-counting barrier (one atomic per CTA), for 148 / 296 co-resident CTAs.
#include <cooperative_groups.h>

#include <cstdio>

namespace cg = cooperative_groups;

__global__ void cg_sync_kernel(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc += 1e-9 * i;
    g.sync();
  }
  if (acc == -1) out[0] = acc;
}

__device__ __forceinline__ void bar_grid(unsigned* count, volatile unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gg = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0u;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == gg) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void bar_kernel(int iters, unsigned* bar, double* out) {
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc += 1e-9 * i;
    bar_grid(bar, bar + 1);
  }
  if (acc == -1) out[0] = acc;
}

int main() {
  double* d;
  unsigned* bar;
  cudaMalloc(&d, 64);
  cudaMalloc(&bar, 64);
  cudaMemset(bar, 0, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int grid : {16, 64, 148, 296}) {
    for (int which = 0; which < 2; ++which) {
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (which == 0) {
          int it = iters;
          void* args[] = {(void*)&it, (void*)&d};
          cudaLaunchCooperativeKernel((void*)cg_sync_kernel, dim3(grid), dim3(256), args, 0, 0);
        } else {
          int it = iters;
          void* args[] = {(void*)&it, (void*)&bar, (void*)&d};
          cudaLaunchCooperativeKernel((void*)bar_kernel, dim3(grid), dim3(256), args, 0, 0);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("{\"barrier\":\"%s\",\"ctas\":%d,\"us_per_barrier\":%.3f,\"err\":\"%s\"}\n",
             which == 0 ? "cg_grid_sync" : "generation_counter", grid, 1000.0 * ms / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
