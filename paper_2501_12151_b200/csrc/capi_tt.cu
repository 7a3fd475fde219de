// extern "C" boundary, part 2: device-resident trains, TT algebra, dense
// factorizations and the AMEn solve (include/qtt.h).
#include <climits>
#include <cmath>
#include <vector>
#include <cstring>
#include <cstdio>
#include <string>

#include "../../include/qtt.h"
#include "amen.cuh"
#include "contract.cuh"
#include "cross.cuh"
#include "linalg.cuh"
#include "sweep.cuh"
#include "capi_internal.cuh"

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return QTT_OK;
  } catch (const qtt::Error& e) {
    return qtt::capi_guard_store(e.what(), e.code);
  } catch (const std::bad_alloc& e) {
    return qtt::capi_guard_store(e.what(), QTT_ERR_CAPACITY);
  } catch (const std::exception& e) {
    return qtt::capi_guard_store(e.what(), QTT_ERR_CUDA);
  }
}

qtt::Ctx& C(qtt_ctx* c) {
  if (!c) throw qtt::Error(QTT_ERR_ARG, "null qtt_ctx");
  QTT_CUDA(cudaSetDevice(c->impl.device));
  return c->impl;
}

const qtt::Train& T(const qtt_train* t) {
  if (!t) throw qtt::Error(QTT_ERR_ARG, "null qtt_train");
  return t->t;
}

void check_chain(const qtt::Train& t) {
  if (t.cores.empty()) throw qtt::Error(QTT_ERR_SHAPE, "a tensor train needs at least one core");
  if (t.cores.front().r0 != 1 || t.cores.back().r1 != 1)
    throw qtt::Error(QTT_ERR_SHAPE, "boundary ranks must be 1");
  for (size_t k = 0; k + 1 < t.cores.size(); ++k)
    if (t.cores[k].r1 != t.cores[k + 1].r0)
      throw qtt::Error(QTT_ERR_SHAPE, "rank mismatch between cores " + std::to_string(k) + " and " +
                                          std::to_string(k + 1));
}

qtt_train* wrap(qtt::Train&& t) {
  auto* h = new qtt_train;
  h->t = std::move(t);
  return h;
}

qtt::DBuf up(const double* h, long long n, cudaStream_t s) {
  qtt::DBuf b(n, s);
  b.upload(h, n);
  return b;
}

}  // namespace

extern "C" {

int qtt_train_upload(qtt_ctx* ctx, int order, int core_ndim, const int64_t* shape, const double* data,
                     qtt_train** out) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (order < 1) throw qtt::Error(QTT_ERR_SHAPE, "a tensor train needs at least one core");
    if (core_ndim != 3 && core_ndim != 4) throw qtt::Error(QTT_ERR_ARG, "core_ndim must be 3 or 4");
    qtt::Train t;
    t.is_op = core_ndim == 4;
    long long off = 0;
    for (int k = 0; k < order; ++k) {
      const int64_t* s = shape + (long long)k * core_ndim;
      for (int d = 0; d < core_ndim; ++d)
        if (s[d] < 1 || s[d] > (1LL << 31)) throw qtt::Error(QTT_ERR_SHAPE, "invalid core shape");
      qtt::Core core = core_ndim == 4 ? qtt::make_core(c, (int)s[0], (int)s[1], (int)s[2], (int)s[3])
                                      : qtt::make_core(c, (int)s[0], (int)s[1], 1, (int)s[2]);
      core.d.upload(data + off, core.numel());
      off += core.numel();
      t.cores.push_back(std::move(core));
    }
    check_chain(t);
    *out = wrap(std::move(t));
  });
}

int qtt_train_info(const qtt_train* t, int* order, int* core_ndim, int64_t* numel) {
  return guarded([&] {
    const qtt::Train& tr = T(t);
    if (order) *order = tr.order();
    if (core_ndim) *core_ndim = tr.is_op ? 4 : 3;
    if (numel) *numel = tr.numel();
  });
}

int qtt_train_shape(const qtt_train* t, int64_t* shape) {
  return guarded([&] {
    const qtt::Train& tr = T(t);
    long long i = 0;
    for (auto& c : tr.cores) {
      shape[i++] = c.r0;
      shape[i++] = c.m;
      if (tr.is_op) shape[i++] = c.n;
      shape[i++] = c.r1;
    }
  });
}

int qtt_train_download(qtt_ctx* ctx, const qtt_train* t, double* data) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    long long off = 0;
    for (auto& core : T(t).cores) {
      core.d.download(data + off, core.numel());
      off += core.numel();
    }
    c.sync();
  });
}

int qtt_train_load_qtt1(qtt_ctx* ctx, const char* path, int* is_operator, qtt_train** out) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (!path || !out) throw qtt::Error(QTT_ERR_ARG, "null path/out");
    const std::string p(path);
    FILE* fh = std::fopen(path, "rb");
    if (!fh) throw qtt::Error(QTT_ERR_ARG, p + ": cannot open");
    std::vector<unsigned char> data;
    {
      unsigned char buf[1 << 16];
      size_t got;
      while ((got = std::fread(buf, 1, sizeof(buf), fh)) > 0) data.insert(data.end(), buf, buf + got);
      std::fclose(fh);
    }
    auto u32 = [&](size_t off) {
      return (uint32_t)data[off] | ((uint32_t)data[off + 1] << 8) | ((uint32_t)data[off + 2] << 16) |
             ((uint32_t)data[off + 3] << 24);
    };
    if (data.size() < 9 || std::memcmp(data.data(), "QTT1", 4) != 0)
      throw qtt::Error(QTT_ERR_FORMAT, p + ": not a QTT1 container (bad magic)");
    const unsigned char kind = data[4];
    if (kind != 'V' && kind != 'O') throw qtt::Error(QTT_ERR_FORMAT, p + ": unknown kind tag");
    const uint32_t count = u32(5);
    size_t off = 9;
    qtt::Train t;
    t.is_op = kind == 'O';
    for (uint32_t k = 0; k < count; ++k) {
      if (off + 16 > data.size())
        throw qtt::Error(QTT_ERR_FORMAT, p + ": truncated header of core " + std::to_string(k));
      const uint32_t d0 = u32(off), d1 = u32(off + 4), d2 = u32(off + 8), d3 = u32(off + 12);
      off += 16;
      // untrusted dims: each must fit an int (core shapes are int), and the product is
      // built with overflow checks against the bytes actually left in the file
      if (d0 > (uint32_t)INT_MAX || d1 > (uint32_t)INT_MAX || d2 > (uint32_t)INT_MAX || d3 > (uint32_t)INT_MAX)
        throw qtt::Error(QTT_ERR_SHAPE, p + ": invalid core dims at core " + std::to_string(k));
      const unsigned long long avail = (data.size() - off) / 8;
      unsigned long long size = 1;
      bool fits = true;
      for (uint32_t dk : {d0, d1, d2, d3}) {
        if (dk != 0 && size > avail / dk) fits = false;
        size *= dk;  // (only used when fits)
      }
      if (!fits || size > avail)
        throw qtt::Error(QTT_ERR_FORMAT, p + ": truncated values of core " + std::to_string(k));
      if (d0 < 1 || d1 < 1 || d2 < 1 || d3 < 1 || (!t.is_op && d2 != 1))
        throw qtt::Error(QTT_ERR_SHAPE, p + ": invalid core dims at core " + std::to_string(k));
      qtt::Core core = qtt::make_core(c, (int)d0, (int)d1, (int)d2, (int)d3);
      // little-endian binary64 on a little-endian host: a straight copy (upload is stream-ordered
      // and the host vector outlives it: synchronized below)
      core.d.upload(reinterpret_cast<const double*>(data.data() + off), (long long)size);
      off += 8 * size;
      t.cores.push_back(std::move(core));
    }
    if (off != data.size())
      throw qtt::Error(QTT_ERR_FORMAT, p + ": " + std::to_string(data.size() - off) + " trailing bytes");
    c.sync();
    check_chain(t);
    if (is_operator) *is_operator = t.is_op ? 1 : 0;
    *out = wrap(std::move(t));
  });
}

int qtt_train_save_qtt1(qtt_ctx* ctx, const qtt_train* th, const char* path) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    const qtt::Train& t = T(th);
    std::vector<unsigned char> out;
    auto put32 = [&](uint32_t v) {
      for (int i = 0; i < 4; ++i) out.push_back((unsigned char)((v >> (8 * i)) & 0xff));
    };
    out.insert(out.end(), {'Q', 'T', 'T', '1', (unsigned char)(t.is_op ? 'O' : 'V')});
    put32((uint32_t)t.cores.size());
    for (const auto& k : t.cores) {
      put32((uint32_t)k.r0);
      put32((uint32_t)k.m);
      put32((uint32_t)k.n);
      put32((uint32_t)k.r1);
      const size_t at = out.size();
      out.resize(at + 8 * (size_t)k.numel());
      QTT_CUDA(cudaMemcpyAsync(out.data() + at, k.d.p, 8 * (size_t)k.numel(), cudaMemcpyDeviceToHost, c.stream));
      c.sync();  // (out may reallocate on the next resize)
    }
    FILE* fh = std::fopen(path, "wb");
    if (!fh) throw qtt::Error(QTT_ERR_ARG, std::string(path) + ": cannot open for writing");
    const size_t w = std::fwrite(out.data(), 1, out.size(), fh);
    std::fclose(fh);
    if (w != out.size()) throw qtt::Error(QTT_ERR_ARG, std::string(path) + ": short write");
  });
}

int qtt_train_free(qtt_train* t) {
  return guarded([&] { delete t; });
}

int qtt_orthogonalize_rl(qtt_ctx* ctx, const qtt_train* a, qtt_train** out) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    qtt::Train g = qtt::clone(c, T(a));
    qtt::orthogonalize_rl(c, g);
    c.sync();
    *out = wrap(std::move(g));
  });
}

int qtt_tt_norm(qtt_ctx* ctx, const qtt_train* a, double* out) {
  return guarded([&] { *out = qtt::tt_norm(C(ctx), T(a)); });
}

int qtt_tt_dot(qtt_ctx* ctx, const qtt_train* a, const qtt_train* b, double* out) {
  return guarded([&] {
    const qtt::Train& ta = T(a);
    const qtt::Train& tb = T(b);
    if (ta.order() != tb.order()) throw qtt::Error(QTT_ERR_SHAPE, "mode dims differ");
    for (int k = 0; k < ta.order(); ++k)
      if (ta.cores[k].m * ta.cores[k].n != tb.cores[k].m * tb.cores[k].n)
        throw qtt::Error(QTT_ERR_SHAPE, "mode dims differ");
    *out = qtt::tt_dot(C(ctx), ta, tb);
  });
}

int qtt_tt_round(qtt_ctx* ctx, const qtt_train* a, double rel_tol, int max_rank, qtt_train** out) {
  return guarded([&] {
    if (rel_tol < 0) throw qtt::Error(QTT_ERR_ARG, "rel_tolerance must be >= 0");
    qtt::Ctx& c = C(ctx);
    qtt::Train r = qtt::tt_round(c, T(a), rel_tol, max_rank);
    c.sync();
    *out = wrap(std::move(r));
  });
}

int qtt_tt_apply(qtt_ctx* ctx, const qtt_train* A, const qtt_train* x, qtt_train** out) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    const qtt::Train& ta = T(A);
    const qtt::Train& tx = T(x);
    if (!ta.is_op || tx.is_op || ta.order() != tx.order())
      throw qtt::Error(QTT_ERR_SHAPE, "operator/vector order mismatch");
    for (int k = 0; k < ta.order(); ++k)
      if (ta.cores[k].n != tx.cores[k].m)
        throw qtt::Error(QTT_ERR_SHAPE, "operator col_dims != vector dims");
    qtt::Train y = qtt::tt_apply(c, ta, tx);
    c.sync();
    *out = wrap(std::move(y));
  });
}

int qtt_tt_apply_into(qtt_ctx* ctx, const qtt_train* A, const qtt_train* x, qtt_train* y) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (!y) throw qtt::Error(QTT_ERR_ARG, "null output train");
    const qtt::Train& ta = T(A);
    const qtt::Train& tx = T(x);
    if (!ta.is_op || tx.is_op || y->t.is_op) throw qtt::Error(QTT_ERR_SHAPE, "operator/vector kinds");
    for (int k = 0; k < ta.order() && k < tx.order(); ++k)
      if (ta.cores[k].n != tx.cores[k].m) throw qtt::Error(QTT_ERR_SHAPE, "operator col_dims != vector dims");
    qtt::tt_apply_into(c, ta, tx, y->t);
    c.sync();
  });
}

int qtt_tt_entries(qtt_ctx* ctx, const qtt_train* t, const int32_t* idx, int64_t count, double* out) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    const qtt::Train& tt = T(t);
    if (count < 0) throw qtt::Error(QTT_ERR_ARG, "negative count");
    const int K = tt.order();
    for (int64_t e = 0; e < count; ++e)
      for (int k = 0; k < K; ++k) {
        const int n = tt.cores[k].m * tt.cores[k].n;
        if (idx[e * K + k] < 0 || idx[e * K + k] >= n)
          throw qtt::Error(QTT_ERR_ARG, "digit " + std::to_string(idx[e * K + k]) + " out of range at mode " +
                                            std::to_string(k));
      }
    if (count == 0) return;
    qtt::DBuf di(qtt::cdiv(count * K, 2) + 1, c.stream), dout(count, c.stream);
    QTT_CUDA(cudaMemcpyAsync(di.p, idx, (size_t)count * K * sizeof(int32_t), cudaMemcpyHostToDevice, c.stream));
    qtt::tt_entries(c, tt, reinterpret_cast<const int*>(di.p), count, dout.p);
    dout.download(out, count);
    c.sync();
  });
}

int qtt_tt_to_dense(qtt_ctx* ctx, const qtt_train* t, int64_t total, double* out) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    const qtt::Train& tt = T(t);
    long long prod = 1;
    for (const auto& k : tt.cores) prod *= (long long)k.m * k.n;
    if (prod != total) throw qtt::Error(QTT_ERR_SHAPE, "output size does not match prod(dims)");
    qtt::DBuf d(total, c.stream);
    qtt::tt_full(c, tt, d.p);
    d.download(out, total);
    c.sync();
  });
}

int qtt_matvec_sweep(qtt_ctx* ctx, const qtt_train* A, const qtt_train* x, int split_timing,
                     qtt_train** y_out, double* times) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    const qtt::Train& tx = T(x);
    T(A);
    check_chain(tx);
    qtt_train* Ah = const_cast<qtt_train*>(A);  // only the cached permuted views are added
    qtt::SweepTimes st;
    qtt::Train y = qtt::matvec_sweep(c, Ah->t, tx, times ? &st : nullptr, split_timing != 0);
    c.sync();
    if (times) {
      const double v[7] = {st.prepass_ms, st.sweep_ms, st.k1_ms, st.k2_ms, st.k1_flops, st.k2_flops,
                           st.prepass_flops};
      for (int i = 0; i < 7; ++i) times[i] = v[i];
    }
    if (y_out) *y_out = wrap(std::move(y));
  });
}

int qtt_residual_norm(qtt_ctx* ctx, const qtt_train* A, const qtt_train* x, const qtt_train* f,
                      int method, double* out, int* used_gram) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (method == 1) *out = qtt::residual_norm_gram(c, T(A), T(x), T(f));
    else *out = qtt::residual_norm(c, T(A), T(x), T(f), nullptr);
    if (used_gram) *used_gram = method == 1 ? 1 : 0;
  });
}

int qtt_qr(qtt_ctx* ctx, const double* mat, int rows, int cols, double* q, double* r) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (rows < 1 || cols < 1) throw qtt::Error(QTT_ERR_SHAPE, "empty matrix");
    const int k = std::min(rows, cols);
    auto dm = up(mat, (long long)rows * cols, c.stream);
    qtt::DBuf dq(q ? (long long)rows * k : 0, c.stream), dr(r ? (long long)k * cols : 0, c.stream);
    qtt::qr(c, qtt::crowmajor(dm.p, rows, cols), q ? qtt::rowmajor(dq.p, rows, k) : qtt::MatView{},
            r ? qtt::rowmajor(dr.p, k, cols) : qtt::MatView{});
    if (q) dq.download(q, dq.n);
    if (r) dr.download(r, dr.n);
    c.sync();
  });
}

int qtt_svd(qtt_ctx* ctx, const double* mat, int rows, int cols, double* u, double* s, double* vt) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (rows < 1 || cols < 1) throw qtt::Error(QTT_ERR_SHAPE, "empty matrix");
    const int k = std::min(rows, cols);
    auto dm = up(mat, (long long)rows * cols, c.stream);
    qtt::DBuf du((long long)rows * k, c.stream), ds(k, c.stream), dv((long long)k * cols, c.stream);
    qtt::svd(c, qtt::crowmajor(dm.p, rows, cols), qtt::rowmajor(du.p, rows, k), ds.p,
             qtt::rowmajor(dv.p, k, cols));
    if (u) du.download(u, du.n);
    if (s) ds.download(s, ds.n);
    if (vt) dv.download(vt, dv.n);
    c.sync();
  });
}

int qtt_rank_for_tolerance(const double* s, int n, double delta, int* out) {
  return guarded([&] { *out = qtt::rank_for_tolerance(s, n, delta); });
}

int qtt_amen_solve(qtt_ctx* ctx, const qtt_train* A, const qtt_train* f, const qtt_train* x0,
                   const qtt_amen_params* prm, const double* draws, int64_t n_draws, qtt_train** x_out,
                   qtt_amen_report* rep, int32_t* rank_hist, double* res_hist) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    const qtt::Train& ta = T(A);
    const qtt::Train& tf = T(f);
    if (!ta.is_op) throw qtt::Error(QTT_ERR_SHAPE, "A must be a TT linear operator");
    if (ta.order() != tf.order()) throw qtt::Error(QTT_ERR_SHAPE, "operator/rhs order mismatch");
    for (int k = 0; k < ta.order(); ++k) {
      if (ta.cores[k].m != ta.cores[k].n) throw qtt::Error(QTT_ERR_SHAPE, "A is not square");
      if (ta.cores[k].n != tf.cores[k].m)
        throw qtt::Error(QTT_ERR_SHAPE, "operator columns do not match f dims");
    }
    if (x0) {
      const qtt::Train& tx = T(x0);
      if (tx.order() != tf.order()) throw qtt::Error(QTT_ERR_SHAPE, "x0 dims do not match f");
      for (int k = 0; k < tf.order(); ++k)
        if (tx.cores[k].m != tf.cores[k].m) throw qtt::Error(QTT_ERR_SHAPE, "x0 dims do not match f");
    }
    qtt::AmenParams p;
    p.residual_tol = prm->residual_tol;
    p.max_sweeps = prm->max_sweeps;
    p.enrichment_rank = prm->enrichment_rank;
    p.local_iterative = prm->local_iterative;
    p.direct_dim_cap = prm->direct_dim_cap;
    p.local_iter_cap = prm->local_iter_cap;
    p.round_tol = prm->round_tol;
    p.round_max_rank = prm->round_max_rank;
    p.stagnation_strikes = prm->stagnation_strikes;
    p.fused_cg = prm->fused_cg;
    qtt::DrawStream ds;
    ds.p = draws;
    ds.n = n_draws;
    qtt::AmenResult res;
    qtt_train* Ah = const_cast<qtt_train*>(A);
    qtt::Train x = qtt::amen_solve(c, Ah->t, tf, x0 ? &T(x0) : nullptr, p, ds, res);
    c.sync();
    rep->converged = res.converged ? 1 : 0;
    rep->sweeps_used = res.sweeps_used;
    rep->final_relative_residual = res.final_residual;
    rep->certifications_gram = res.certifications_gram;
    rep->certifications_exact = res.certifications_exact;
    rep->draws_used = ds.pos;
    const int K = ta.order();
    for (int s = 0; s < res.sweeps_used && s < p.max_sweeps; ++s) {
      if (rank_hist)
        for (int j = 0; j <= K; ++j) rank_hist[(long long)s * (K + 1) + j] = res.rank_history[s][j];
      if (res_hist) res_hist[s] = res.residual_history[s];
    }
    *x_out = wrap(std::move(x));
  });
}

int qtt_maxvol(qtt_ctx* ctx, const double* mat, int rows, int cols, int qr, double tol, int max_iters,
               int32_t* piv, double* b, int* status) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (!mat || !piv || rows < 1 || cols < 1) throw qtt::Error(QTT_ERR_ARG, "maxvol: bad arguments");
    if (rows < cols) throw qtt::Error(QTT_ERR_SHAPE, "maxvol needs a tall matrix");
    auto dm = up(mat, (long long)rows * cols, c.stream);
    qtt::DBuf q;
    const double* A = dm.p;
    if (qr) {  // thin Q (rows x cols), numpy.linalg.qr conventions
      q.alloc((long long)rows * cols, c.stream);
      qtt::qr(c, qtt::crowmajor(dm.p, rows, cols), qtt::rowmajor(q.p, rows, cols), qtt::MatView{});
      A = q.p;
    }
    qtt::DBuf B((long long)rows * cols, c.stream);
    int* dpiv = nullptr;
    QTT_CUDA(cudaMallocAsync((void**)&dpiv, sizeof(int) * (cols + 1), c.stream));
    const int st = qtt::maxvol(c, A, rows, cols, tol, max_iters, B.p, dpiv, dpiv + cols);
    std::vector<int> hp(cols);
    QTT_CUDA(cudaMemcpyAsync(hp.data(), dpiv, sizeof(int) * cols, cudaMemcpyDeviceToHost, c.stream));
    if (b) B.download(b, B.n);
    c.sync();
    cudaFreeAsync(dpiv, c.stream);
    for (int i = 0; i < cols; ++i) piv[i] = hp[i];
    if (status) *status = st;
  });
}

int qtt_amen_step(qtt_ctx* ctx, const qtt_train* A, const qtt_train* f, const qtt_amen_params* prm,
                  int sweep, int k, int forward, double lam_max, double f_norm, int n_in,
                  const double* const* in, const int64_t* in_dims, qtt_train** out, double* lam,
                  int* rank, int* iters) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (!A || !f || !prm || !in || !in_dims || !out) throw qtt::Error(QTT_ERR_ARG, "null argument");
    if (!T(A).is_op) throw qtt::Error(QTT_ERR_SHAPE, "A must be a TT linear operator");
    if (n_in != 11) throw qtt::Error(QTT_ERR_ARG, "qtt_amen_step takes 11 state arrays");
    std::vector<qtt::HostArray> st(n_in);
    for (int i = 0; i < n_in; ++i) {
      for (int d = 0; d < 3; ++d)
        if (in_dims[3 * i + d] < 1 || in_dims[3 * i + d] > INT_MAX) throw qtt::Error(QTT_ERR_SHAPE, "bad state dims");
      st[i].d0 = (int)in_dims[3 * i];
      st[i].d1 = (int)in_dims[3 * i + 1];
      st[i].d2 = (int)in_dims[3 * i + 2];
      st[i].v.assign(in[i], in[i] + (size_t)st[i].d0 * st[i].d1 * st[i].d2);
    }
    qtt::AmenParams p;
    p.residual_tol = prm->residual_tol;
    p.max_sweeps = prm->max_sweeps;
    p.enrichment_rank = prm->enrichment_rank;
    p.local_iterative = prm->local_iterative;
    p.direct_dim_cap = prm->direct_dim_cap;
    p.local_iter_cap = prm->local_iter_cap;
    p.round_tol = prm->round_tol;
    p.round_max_rank = prm->round_max_rank;
    p.stagnation_strikes = prm->stagnation_strikes;
    p.fused_cg = prm->fused_cg;
    std::vector<qtt::HostArray> res;
    qtt::StepInfo info;
    qtt_train* Ah = const_cast<qtt_train*>(A);
    qtt::amen_core_step(c, Ah->t, T(f), p, sweep, k, forward != 0, lam_max, f_norm, st, res, info);
    qtt::Train b;  // unchained bundle of the step's outputs
    for (auto& h : res) {
      qtt::Core core = qtt::make_core(c, h.d0, h.d1, 1, h.d2);
      core.d.upload(h.v.data(), core.numel());
      b.cores.push_back(std::move(core));
    }
    c.sync();
    if (lam) *lam = info.lam;
    if (rank) *rank = info.rank;
    if (iters) *iters = info.iters;
    *out = wrap(std::move(b));
  });
}

int qtt_local_solve(qtt_ctx* ctx, const double* phil, const double* A, const double* phir,
                    const double* rhs, const double* prev, int rl, int R0, int m, int R1, int rr,
                    int iterative, int direct_dim_cap, double residual_tol, int iter_cap, int fused_cg,
                    double* u, double* lam, int* iterations) {
  return guarded([&] {
    qtt::Ctx& c = C(ctx);
    if (rl < 1 || R0 < 1 || m < 1 || R1 < 1 || rr < 1) throw qtt::Error(QTT_ERR_SHAPE, "bad local shape");
    cudaStream_t s = c.stream;
    const long long dim = (long long)rl * m * rr;
    auto dl = up(phil, (long long)rl * R0 * rl, s);
    auto dA = up(A, (long long)R0 * m * m * R1, s);
    auto dr = up(phir, (long long)rr * R1 * rr, s);
    auto db = up(rhs, dim, s);
    auto dp = up(prev, dim, s);
    qtt::DBuf Ap((long long)R0 * m * m * R1, s);
    qtt::permute_op_core(dA.p, R0, m, m, R1, Ap.p, nullptr, s);
    qtt::LocalSystem L{dl.p, rl, R0, rl, dA.p, Ap.p, R0, m, m, R1, dr.p, rr, R1, rr};
    qtt::AmenParams p;
    p.local_iterative = iterative;
    p.direct_dim_cap = direct_dim_cap;
    p.residual_tol = residual_tol;
    p.local_iter_cap = iter_cap;
    p.fused_cg = fused_cg;
    double l = 0;
    int it = 0;
    qtt::DBuf du = qtt::solve_local_system(c, L, db.p, dp.p, p, 0, 0, l, it, false);
    du.download(u, dim);
    c.sync();
    if (lam) *lam = l;
    if (iterations) *iterations = it;
  });
}

}  // extern "C"
