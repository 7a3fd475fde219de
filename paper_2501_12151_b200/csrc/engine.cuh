// Engine context: one CUDA stream + a stream-ordered memory pool per context
// (re-entrant per handle, no global mutable state; SURVEY.md 8b "Threading").
#pragma once
#include <vector>

#include "common.cuh"

namespace qtt {

struct Stats {
  long long launches = 0;       // kernel launches issued by this engine (all kinds)
  long long k1_calls = 0;       // local matvec (K1) invocations
  double k1_flops = 0, k1_ms = 0;
  long long env_calls = 0;      // environment updates (K2)
  double env_flops = 0, env_ms = 0;
  long long cg_iters = 0, cg_solves = 0, chol_solves = 0;
  long long svd_calls = 0, qr_calls = 0;
  long long sweeps = 0, certifications = 0;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool profiling = false;
  Stats stats;
  // pinned host staging for small scalar readbacks
  double* pinned = nullptr;
  size_t pinned_n = 0;
  std::vector<cudaEvent_t> ev_pool;
  // deterministic-reduction scratch (linalg.cu) and small device flags
  double* red_partial = nullptr;   // 1024 doubles
  unsigned* red_counter = nullptr; // 1 counter
  int* flags = nullptr;            // 64 ints (Cholesky info, CG done, ...)
  double* scal = nullptr;          // 256 device scalars
  explicit Ctx(int dev);
  ~Ctx();
  double* host_scalars(size_t n);
  void sync() { QTT_CUDA(cudaStreamSynchronize(stream)); }
};

// Stream-ordered device buffer (cudaMallocAsync on the context stream).
struct DBuf {
  double* p = nullptr;
  long long n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(long long count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(long long count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count > 0) QTT_CUDA(cudaMallocAsync((void**)&p, (size_t)count * sizeof(double), st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  void upload(const double* h, long long count) {
    QTT_CUDA(cudaMemcpyAsync(p, h, (size_t)count * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  void download(double* h, long long count) const {
    QTT_CUDA(cudaMemcpyAsync(h, p, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
};

}  // namespace qtt
