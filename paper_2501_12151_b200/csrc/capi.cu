// extern "C" boundary (include/qtt.h).  Every entry point converts exceptions to
// status codes and records a thread-local message for qtt_last_error().
#include <atomic>
#include <cstring>
#include <string>

#include "../../include/qtt.h"
#include "capi_internal.cuh"
#include "contract.cuh"
#include "engine.cuh"

namespace qtt {

Ctx::Ctx(int dev) : device(dev) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw Error(QTT_ERR_CUDA, "no CUDA device available: the QTT engine has no CPU fallback");
  if (dev < 0 || dev >= count) throw Error(QTT_ERR_ARG, "device index out of range");
  QTT_CUDA(cudaSetDevice(dev));
  QTT_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  QTT_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thresh = UINT64_MAX;  // keep freed blocks cached in the pool
  QTT_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
  QTT_CUDA(cudaMalloc((void**)&red_partial, 1024 * sizeof(double)));
  QTT_CUDA(cudaMalloc((void**)&red_counter, 64 * sizeof(unsigned)));
  QTT_CUDA(cudaMemset(red_counter, 0, 64 * sizeof(unsigned)));
  QTT_CUDA(cudaMalloc((void**)&flags, 64 * sizeof(int)));
  QTT_CUDA(cudaMemset(flags, 0, 64 * sizeof(int)));
  QTT_CUDA(cudaMalloc((void**)&scal, 256 * sizeof(double)));
}

Ctx::~Ctx() {
  l2_flush.release();
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
  if (pinned) cudaFreeHost(pinned);
  if (red_partial) cudaFree(red_partial);
  if (red_counter) cudaFree(red_counter);
  if (flags) cudaFree(flags);
  if (scal) cudaFree(scal);
  for (auto ev : ev_pool) cudaEventDestroy(ev);
}

static std::atomic<long long> g_launches{0};
long long launch_count() { return g_launches.load(); }
void count_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void Ctx::phase(int ph) {
  if (!phase_sync) return;
  sync();
  const double t = std::chrono::duration<double, std::milli>(
                       std::chrono::steady_clock::now().time_since_epoch()).count();
  if (phase_t0 >= 0) stats.phase_ms[phase_cur] += t - phase_t0;
  phase_t0 = t;
  phase_cur = ph;
}

void Ctx::prof_flush() {
  if (prof.pending.empty()) return;
  sync();
  for (auto& r : prof.pending) {
    if (!r.keep) continue;
    float ms = 0;
    QTT_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    if (r.kind == 0) { stats.k1_ms += ms; stats.k1_timed_flops += r.flops; }
    else { stats.env_ms += ms; stats.env_timed_flops += r.flops; }
  }
  prof.pending.clear();
  prof.next = 0;
}

double* Ctx::host_scalars(size_t n) {
  if (n > pinned_n) {
    if (pinned) QTT_CUDA(cudaFreeHost(pinned));
    pinned_n = std::max<size_t>(n, 4096);
    QTT_CUDA(cudaMallocHost((void**)&pinned, pinned_n * sizeof(double)));
  }
  return pinned;
}

}  // namespace qtt

namespace {

thread_local std::string g_last_error;

}  // namespace

int qtt::capi_guard_store(const char* what, int code) {
  g_last_error = what;
  return code;
}

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return QTT_OK;
  } catch (const qtt::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("host allocation failed: ") + e.what();
    return QTT_ERR_CAPACITY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return QTT_ERR_CUDA;
  }
}

void check_ctx(qtt_ctx* c) {
  if (!c) throw qtt::Error(QTT_ERR_ARG, "null qtt_ctx");
  QTT_CUDA(cudaSetDevice(c->impl.device));
}

void check_dims(std::initializer_list<int> dims) {
  for (int d : dims)
    if (d <= 0) throw qtt::Error(QTT_ERR_SHAPE, "all core dimensions must be positive");
}

long long prod(std::initializer_list<long long> v) {
  long long p = 1;
  for (auto x : v) p *= x;
  return p;
}

// Upload a host array into a fresh stream-ordered buffer.
qtt::DBuf up(const double* h, long long n, cudaStream_t s) {
  qtt::DBuf b(n, s);
  b.upload(h, n);
  return b;
}

}  // namespace

extern "C" {

int qtt_version(void) { return 1; }

const char* qtt_last_error(void) { return g_last_error.c_str(); }

int qtt_ctx_create(int device, qtt_ctx** out) {
  return guarded([&] {
    if (!out) throw qtt::Error(QTT_ERR_ARG, "null output pointer");
    *out = new qtt_ctx(device);
  });
}

int qtt_ctx_destroy(qtt_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

int qtt_ctx_synchronize(qtt_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->impl.sync();
  });
}

void* qtt_ctx_stream(qtt_ctx* ctx) { return ctx ? (void*)ctx->impl.stream : nullptr; }

int qtt_ctx_set_profiling(qtt_ctx* ctx, int on) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->impl.profiling = (on & 1) != 0;
    ctx->impl.phase_sync = (on & 2) != 0;
  });
}

int qtt_ctx_flush_l2(qtt_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    qtt::Ctx& c = ctx->impl;
    const long long n = 256LL << 20;  // 256 MiB > 126 MB L2
    if (c.l2_flush.n < n / 8) c.l2_flush.alloc(n / 8, c.stream);
    QTT_CUDA(cudaMemsetAsync(c.l2_flush.p, 0, n, c.stream));
  });
}

int64_t qtt_launch_count(void) { return qtt::launch_count(); }

int qtt_ctx_get_stats(qtt_ctx* ctx, qtt_stats* o) {
  return guarded([&] {
    check_ctx(ctx);
    const qtt::Stats& s = ctx->impl.stats;
    o->launches = s.launches;
    o->k1_calls = s.k1_calls;
    o->k1_flops = s.k1_flops;
    o->k1_ms = s.k1_ms;
    o->env_calls = s.env_calls;
    o->env_flops = s.env_flops;
    o->env_ms = s.env_ms;
    o->k1_timed_flops = s.k1_timed_flops;
    o->env_timed_flops = s.env_timed_flops;
    o->launches = qtt::launch_count();
    for (int i = 0; i < 10; ++i) o->phase_ms[i] = s.phase_ms[i];
    o->cg_iters = s.cg_iters;
    o->cg_solves = s.cg_solves;
    o->chol_solves = s.chol_solves;
    o->svd_calls = s.svd_calls;
    o->qr_calls = s.qr_calls;
    o->sweeps = s.sweeps;
    o->certifications = s.certifications;
  });
}

int qtt_ctx_reset_stats(qtt_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->impl.stats = qtt::Stats();
    ctx->impl.trace.clear();
  });
}

int qtt_ctx_trace(qtt_ctx* ctx, int32_t* out, int64_t cap, int64_t* n) {
  return guarded([&] {
    check_ctx(ctx);
    const auto& t = ctx->impl.trace;
    *n = (int64_t)t.size();
    const int64_t k = std::min<int64_t>(cap, (int64_t)t.size());
    for (int64_t i = 0; i < k; ++i) {
      const auto& r = t[i];
      const int32_t v[11] = {r.sweep, r.core, r.rl, r.m, r.rr, r.zl, r.zr, r.R0, r.R1, r.path, r.iters};
      for (int j = 0; j < 11; ++j) out[i * 11 + j] = v[j];
    }
  });
}


int qtt_local_matvec(qtt_ctx* ctx, const double* phil, const double* A, const double* phir,
                     const double* x, int rX, int Ra, int rU, int m, int n, int Rb, int rY, int rV,
                     double* y) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, Ra, rU, m, n, Rb, rY, rV});
    cudaStream_t s = ctx->impl.stream;
    auto dphil = up(phil, prod({rX, Ra, rU}), s);
    auto dA = up(A, prod({Ra, m, n, Rb}), s);
    auto dphir = up(phir, prod({rY, Rb, rV}), s);
    auto dx = up(x, prod({rU, n, rV}), s);
    qtt::DBuf Ap(prod({Ra, m, n, Rb}), s), dy(prod({rX, m, rY}), s);
    qtt::permute_op_core(dA.p, Ra, m, n, Rb, Ap.p, nullptr, s);
    long long need = qtt::local_matvec_scratch(rX, Ra, rU, m, n, Rb, rY, rV);
    qtt::DBuf sc(need + prod({rX * m, rY, 64}), s);
    qtt::local_matvec(dphil.p, rX, Ra, rU, Ap.p, m, n, Rb, dphir.p, rY, rV, dx.p, dy.p, 1.0, 0.0,
                      {sc.p, sc.n}, s);
    dy.download(y, dy.n);
    ctx->impl.sync();
  });
}

int qtt_env_left(qtt_ctx* ctx, const double* phi, const double* bra, const double* A,
                 const double* ket, int rX, int RA, int rY, int m, int n, int RB, int rU, int rZ,
                 double* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, RA, rY, m, n, RB, rU, rZ});
    cudaStream_t s = ctx->impl.stream;
    auto dphi = up(phi, prod({rX, RA, rY}), s);
    auto dbra = up(bra, prod({rX, m, rU}), s);
    auto dA = up(A, prod({RA, m, n, RB}), s);
    auto dket = up(ket, prod({rY, n, rZ}), s);
    qtt::DBuf Ap(prod({RA, m, n, RB}), s), dout(prod({rU, RB, rZ}), s);
    qtt::permute_op_core(dA.p, RA, m, n, RB, Ap.p, nullptr, s);
    long long need = qtt::env_left_scratch(rX, RA, rY, m, n, RB, rZ, rU);
    qtt::DBuf sc(need + prod({rU, RB * rZ, 64}), s);
    qtt::env_left(dphi.p, rX, RA, rY, dbra.p, rU, Ap.p, m, n, RB, dket.p, rZ, dout.p, {sc.p, sc.n}, s);
    dout.download(out, dout.n);
    ctx->impl.sync();
  });
}

int qtt_env_right(qtt_ctx* ctx, const double* phi, const double* bra, const double* A,
                  const double* ket, int rX, int RA, int rZ, int m, int n, int Ra, int rB, int rY,
                  double* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, RA, rZ, m, n, Ra, rB, rY});
    cudaStream_t s = ctx->impl.stream;
    auto dphi = up(phi, prod({rX, RA, rZ}), s);
    auto dbra = up(bra, prod({rB, m, rX}), s);
    auto dA = up(A, prod({Ra, m, n, RA}), s);
    auto dket = up(ket, prod({rY, n, rZ}), s);
    qtt::DBuf Aq(prod({Ra, m, n, RA}), s), dout(prod({rB, Ra, rY}), s);
    qtt::permute_op_core(dA.p, Ra, m, n, RA, nullptr, Aq.p, s);
    long long need = qtt::env_right_scratch(rX, RA, rZ, m, n, Ra, rY, rB);
    qtt::DBuf sc(need + prod({rB, Ra * rY, 64}), s);
    qtt::env_right(dphi.p, rX, RA, rZ, dbra.p, rB, Aq.p, m, n, Ra, dket.p, rY, dout.p, {sc.p, sc.n}, s);
    dout.download(out, dout.n);
    ctx->impl.sync();
  });
}

int qtt_psi_left(qtt_ctx* ctx, const double* psi, const double* bra, const double* f, int rX,
                 int rF, int m, int rU, int rG, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, rF, m, rU, rG});
    cudaStream_t s = ctx->impl.stream;
    auto dpsi = up(psi, prod({rX, rF}), s);
    auto dbra = up(bra, prod({rX, m, rU}), s);
    auto df = up(f, prod({rF, m, rG}), s);
    qtt::DBuf dout(prod({rU, rG}), s), sc(prod({rX, m, rG}) + prod({rU, rG, 64}), s);
    qtt::psi_left(dpsi.p, rX, rF, dbra.p, m, rU, df.p, rG, dout.p, {sc.p, sc.n}, s);
    dout.download(out, dout.n);
    ctx->impl.sync();
  });
}

int qtt_psi_right(qtt_ctx* ctx, const double* psi, const double* bra, const double* f, int rX,
                  int rG, int rU, int m, int rF, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, rG, rU, m, rF});
    cudaStream_t s = ctx->impl.stream;
    auto dpsi = up(psi, prod({rX, rG}), s);
    auto dbra = up(bra, prod({rU, m, rX}), s);
    auto df = up(f, prod({rF, m, rG}), s);
    qtt::DBuf dout(prod({rU, rF}), s), sc(prod({rF, m, rX}) + prod({rU, rF, 64}), s);
    qtt::psi_right(dpsi.p, rX, rG, dbra.p, rU, m, df.p, rF, dout.p, {sc.p, sc.n}, s);
    dout.download(out, dout.n);
    ctx->impl.sync();
  });
}

int qtt_local_rhs(qtt_ctx* ctx, const double* psil, const double* f, const double* psir, int rX,
                  int rF, int m, int rG, int rY, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, rF, m, rG, rY});
    cudaStream_t s = ctx->impl.stream;
    auto dl = up(psil, prod({rX, rF}), s);
    auto df = up(f, prod({rF, m, rG}), s);
    auto dr = up(psir, prod({rY, rG}), s);
    qtt::DBuf dout(prod({rX, m, rY}), s), sc(prod({rX, m, rG}) + prod({rX * m, rY, 64}), s);
    qtt::local_rhs(dl.p, rX, rF, df.p, m, rG, dr.p, rY, dout.p, {sc.p, sc.n}, s);
    dout.download(out, dout.n);
    ctx->impl.sync();
  });
}

int qtt_local_dense(qtt_ctx* ctx, const double* phil, const double* A, const double* phir, int rX,
                    int Ra, int rU, int m, int n, int Rb, int rY, int rV, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, Ra, rU, m, n, Rb, rY, rV});
    cudaStream_t s = ctx->impl.stream;
    auto dl = up(phil, prod({rX, Ra, rU}), s);
    auto dA = up(A, prod({Ra, m, n, Rb}), s);
    auto dr = up(phir, prod({rY, Rb, rV}), s);
    qtt::DBuf dout(prod({rX, m, rY}) * prod({rU, n, rV}), s);
    qtt::DBuf sc(qtt::local_dense_scratch(rX, Ra, rU, m, n, Rb), s);
    qtt::local_dense(dl.p, rX, Ra, rU, dA.p, m, n, Rb, dr.p, rY, rV, dout.p, {sc.p, sc.n}, s);
    dout.download(out, dout.n);
    ctx->impl.sync();
  });
}

int qtt_local_diag(qtt_ctx* ctx, const double* phil, const double* A, const double* phir, int rX,
                   int Ra, int m, int Rb, int rY, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, Ra, m, Rb, rY});
    cudaStream_t s = ctx->impl.stream;
    auto dl = up(phil, prod({rX, Ra, rX}), s);
    auto dA = up(A, prod({Ra, m, m, Rb}), s);
    auto dr = up(phir, prod({rY, Rb, rY}), s);
    qtt::DBuf dout(prod({rX, m, rY}), s), sc(prod({rX, m, Rb}), s);
    qtt::local_diag(dl.p, rX, Ra, dA.p, m, Rb, dr.p, rY, dout.p, {sc.p, sc.n}, s);
    dout.download(out, dout.n);
    ctx->impl.sync();
  });
}

int qtt_mixed_residual(qtt_ctx* ctx, const double* psil, const double* f, const double* psir,
                       const double* phil, const double* A, const double* u, const double* phir,
                       int rX, int rF, int rG, int rY, int Ra, int rU, int m, int n, int Rb, int rV,
                       double* out) {
  return guarded([&] {
    check_ctx(ctx);
    check_dims({rX, rF, rG, rY, Ra, rU, m, n, Rb, rV});
    cudaStream_t s = ctx->impl.stream;
    auto dpl = up(psil, prod({rX, rF}), s);
    auto df = up(f, prod({rF, m, rG}), s);
    auto dpr = up(psir, prod({rY, rG}), s);
    auto dl = up(phil, prod({rX, Ra, rU}), s);
    auto dA = up(A, prod({Ra, m, n, Rb}), s);
    auto du = up(u, prod({rU, n, rV}), s);
    auto dr = up(phir, prod({rY, Rb, rV}), s);
    qtt::DBuf Ap(prod({Ra, m, n, Rb}), s), dout(prod({rX, m, rY}), s);
    qtt::permute_op_core(dA.p, Ra, m, n, Rb, Ap.p, nullptr, s);
    long long need = std::max(qtt::local_matvec_scratch(rX, Ra, rU, m, n, Rb, rY, rV),
                              prod({rX, m, rG})) + prod({rX * m, rY, 64});
    qtt::DBuf sc(need, s);
    qtt::local_rhs(dpl.p, rX, rF, df.p, m, rG, dpr.p, rY, dout.p, {sc.p, sc.n}, s);
    qtt::local_matvec(dl.p, rX, Ra, rU, Ap.p, m, n, Rb, dr.p, rY, rV, du.p, dout.p, -1.0, 1.0,
                      {sc.p, sc.n}, s);
    dout.download(out, dout.n);
    ctx->impl.sync();
  });
}

}  // extern "C"
