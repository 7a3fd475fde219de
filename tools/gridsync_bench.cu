// Cost of one grid-wide barrier in a persistent cooperative kernel (148 CTAs x 384 threads,
// the CG kernel's launch shape):  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/gridsync_bench.cu -o /tmp/gsb && /tmp/gsb
//   mode 0: cooperative_groups grid.sync()
//   mode 1: sense-reversing counter: thread 0 red.release.gpu.add, last arriver flips a flag
//           with st.release.gpu, others poll ld.acquire.gpu (one L2 line each)
//   mode 2: two-level: cluster barrier, one arrival per CTA pair (cooperative + cluster launch),
//           the pair leader polls, cluster barrier
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ unsigned g_count, g_flag;
__device__ unsigned g_flags[1024 * 8];  // mode 3/4: one epoch word per CTA (packed / one per 32-byte sector)

// mode 3/4: no atomics.  Thread 0 publishes the CTA's epoch with st.release.gpu; thread i polls
// CTA i's word with ld.acquire.gpu until it reaches the epoch; block barrier.  The 148 arrivals do
// not serialise on one L2 address as the counter's atomics do.
template <int STRIDE>
__device__ __forceinline__ void bar3(unsigned nblocks, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0)
    asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&g_flags[blockIdx.x * STRIDE]), "r"(epoch) : "memory");
  for (unsigned i = threadIdx.x; i < nblocks; i += blockDim.x) {
    unsigned f;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(f) : "l"(&g_flags[i * STRIDE]) : "memory");
    } while ((int)(f - epoch) < 0);
  }
  __syncthreads();
}

__device__ __forceinline__ void bar1(unsigned nblocks, unsigned& sense) {
  __syncthreads();
  if (threadIdx.x == 0) {
    sense ^= 1u;
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(&g_count) : "memory");
    if (old == nblocks - 1) {
      g_count = 0;
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&g_flag), "r"(sense) : "memory");
    } else {
      unsigned f;
      do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(f) : "l"(&g_flag) : "memory"); } while (f != sense);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void bar2(unsigned nclusters, unsigned& gen) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    const unsigned target = (gen + 1) * nclusters;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&g_count) : "memory");
    unsigned f;
    do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(f) : "l"(&g_count) : "memory"); } while (f < target);
  }
  ++gen;
  cl.sync();
}

__global__ void kern(int iters, int mode, double* sink) {
  unsigned sense = 0;
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    acc = acc * 1.0000001 + 1.0;
    if (mode == 0) cg::this_grid().sync();
    else if (mode == 1) bar1(gridDim.x, sense);
    else if (mode == 3) bar3<1>(gridDim.x, sense);
    else if (mode == 4) bar3<8>(gridDim.x, sense);
    else bar2(gridDim.x / 2, sense);
  }
  if (acc == -1.0) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  for (int mode : {0, 1, 3, 4}) {
    cudaMemset(nullptr, 0, 0);
    {
      void* p = nullptr;
      cudaGetSymbolAddress(&p, g_flags);
      cudaMemset(p, 0, sizeof(unsigned) * 1024 * 8);
    }
    for (int nt : {128, 384}) {
      int iters = 20000;
      void* args[] = {&iters, &mode, &sink};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaLaunchCooperativeKernel((void*)kern, sms, nt, args, 0, 0);  // warm-up
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)kern, sms, nt, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("mode %d grid %d x %d: %.3f us per barrier (%s)\n", mode, sms, nt, ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int nt : {128, 384}) {  // mode 2: clusters of 2
    int iters = 20000, mode = 2;
    unsigned zero = 0;
    cudaMemcpyToSymbol(g_count, &zero, 4);
    void* args[] = {&iters, &mode, &sink};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(nt);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = cudaLaunchKernelExC(&cfg, (void*)kern, args);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("mode 2 grid %d x %d (clusters of 2): %.3f us per barrier (%s / %s)\n", sms, nt, ms * 1e3 / iters,
           cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
