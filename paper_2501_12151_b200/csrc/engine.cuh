// Engine context: one CUDA stream + a stream-ordered memory pool per context
// (re-entrant per handle, no global mutable state; SURVEY.md 8b "Threading").
#pragma once
#include <chrono>
#include <vector>

#include "common.cuh"

namespace qtt {

struct Stats {
  long long launches = 0;       // kernel launches issued by this engine (all kinds)
  long long k1_calls = 0;       // local matvec (K1) invocations
  double k1_flops = 0, k1_ms = 0, k1_timed_flops = 0;
  long long env_calls = 0;      // environment updates (K2)
  double env_flops = 0, env_ms = 0, env_timed_flops = 0;
  long long cg_iters = 0, cg_solves = 0, chol_solves = 0;
  long long svd_calls = 0, qr_calls = 0;
  long long sweeps = 0, certifications = 0;
  // wall time per solver phase (profiling mode syncs at phase boundaries)
  double phase_ms[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
};
enum Phase { PH_OTHER = 0, PH_DIRECT, PH_CG, PH_MIXED, PH_SVD, PH_QR, PH_ENV, PH_CERT, PH_PREPASS, PH_RHS };

// Deferred CUDA-event timing of the contraction kernels (no host sync at record
// time; pending pairs are resolved at the solver's existing sync points).
struct Profiler {
  struct Rec {
    cudaEvent_t a, b;
    int kind;       // 0: K1 local matvec, 1: K2 environment update
    double flops;
    bool keep;
  };
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  std::vector<Rec> pending;
  cudaEvent_t get() {
    if (next == pool.size()) {
      cudaEvent_t e;
      QTT_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[next++];
  }
  ~Profiler() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// One local solve of a sweep (for the CPU-baseline cost model and diagnostics).
struct TraceRec {
  int sweep, core, rl, m, rr, zl, zr, R0, R1, path /*0 direct, 1 cg*/, iters;
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

struct Ctx {
  int device = 0;
  std::vector<TraceRec> trace;
  cudaStream_t stream = nullptr;
  bool profiling = false;   // CUDA-event timing of K1/K2 launches (deferred, no syncs)
  bool phase_sync = false;  // per-phase wall timing (synchronizes at phase boundaries)
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
  Profiler prof;
  DBuf l2_flush;  // scratch written between timed steps (bench L2 flush)
  explicit Ctx(int dev);
  ~Ctx();
  // profiling helpers (no-ops unless profiling): begin returns a record id or -1
  int prof_begin() {
    if (!profiling) return -1;
    Profiler::Rec r{prof.get(), prof.get(), 0, 0.0, true};
    QTT_CUDA(cudaEventRecord(r.a, stream));
    prof.pending.push_back(r);
    return (int)prof.pending.size() - 1;
  }
  void prof_end(int id, int kind, double flops) {
    if (id < 0) return;
    auto& r = prof.pending[id];
    QTT_CUDA(cudaEventRecord(r.b, stream));
    r.kind = kind;
    r.flops = flops;
  }
  void prof_discard(int id) {
    if (id >= 0) prof.pending[id].keep = false;
  }
  // resolve pending records (synchronizes the stream)
  void prof_flush();
  int phase_cur = 0;
  double phase_t0 = -1;
  void phase(int ph);
  double* host_scalars(size_t n);
  void sync() { QTT_CUDA(cudaStreamSynchronize(stream)); }
};



}  // namespace qtt
