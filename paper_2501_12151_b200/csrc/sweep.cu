// One AMEn-style interface sweep without the local solve: the config-4 microbench of
// SURVEY.md 8d.  Right-environment pre-pass (amen.py:300-321 with bra = ket = x,
// _phi_right_step amen.py:114-117), then for k = 0..K-1 the local matvec
// y_k = _local_matvec(phi_L[k], A_k, phi_R[k+1], x_k) (amen.py:134-137) followed by
// phi_L[k+1] = _phi_left_step(phi_L[k], x_k, A_k, x_k) (amen.py:108-111).
// Environments stay in HBM for the whole pass; one scratch arena serves every step.
#include <algorithm>
#include <string>
#include <vector>

#include "contract.cuh"
#include "linalg.cuh"
#include "sweep.cuh"

namespace qtt {
namespace {

struct EnvBuf {
  int b = 1, o = 1, k = 1;
  DBuf d;
};

struct EvPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

double elapsed(const EvPair& e) {
  float ms = 0.f;
  QTT_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
  return ms;
}

}  // namespace

Train matvec_sweep(Ctx& c, Train& A, const Train& x, SweepTimes* t, bool split_timing) {
  const int K = A.order();
  if (x.order() != K || !A.is_op || x.is_op) throw Error(QTT_ERR_SHAPE, "operator/vector order mismatch");
  for (int k = 0; k < K; ++k) {
    const Core &a = A.cores[k], &v = x.cores[k];
    if (a.n != v.m || a.m != v.m)
      throw Error(QTT_ERR_SHAPE, "matvec sweep needs a square operator matching the vector modes (core " +
                                     std::to_string(k) + ")");
  }
  prepare_operator(c, A);
  // one scratch arena, sized for the largest step
  long long need = 0;
  for (int k = 0; k < K; ++k) {
    const Core &a = A.cores[k], &v = x.cores[k];
    // (same per-call margins as the solver's own calls, amen.cu)
    need = std::max(need, env_right_scratch(v.r1, a.r1, v.r1, a.m, a.n, a.r0, v.r0, v.r0) +
                              (long long)v.r0 * a.r0 * v.r0 * 4);
    need = std::max(need, env_left_scratch(v.r0, a.r0, v.r0, a.m, a.n, a.r1, v.r1, v.r1) +
                              (long long)v.r1 * a.r1 * v.r1 * 4);
    need = std::max(need, local_matvec_scratch(v.r0, a.r0, v.r0, a.m, a.n, a.r1, v.r1, v.r1) +
                              (long long)v.r0 * a.m * v.r1 * 8);
  }
  DBuf sc(need, c.stream);
  std::vector<EnvBuf> R(K + 1);
  R[K].d.alloc(1, c.stream);
  fill(c, R[K].d.p, 1, 1.0);
  EnvBuf L;
  L.d.alloc(1, c.stream);
  fill(c, L.d.p, 1, 1.0);

  std::vector<cudaEvent_t> evs;
  auto ev = [&]() {
    cudaEvent_t e;
    QTT_CUDA(cudaEventCreate(&e));
    evs.push_back(e);
    QTT_CUDA(cudaEventRecord(e, c.stream));
    return e;
  };
  const bool timed = t != nullptr;
  EvPair pre, sw;
  std::vector<EvPair> k1, k2;
  if (timed) pre.a = ev();
  for (int k = K - 1; k >= 1; --k) {
    const Core &a = A.cores[k], &v = x.cores[k];
    EnvBuf& o = R[k];
    o.b = v.r0; o.o = a.r0; o.k = v.r0;
    o.d.alloc((long long)o.b * o.o * o.k, c.stream);
    env_right(R[k + 1].d.p, R[k + 1].b, R[k + 1].o, R[k + 1].k, v.d.p, v.r0, A.Aq[k].p, a.m, a.n, a.r0,
              v.d.p, v.r0, o.d.p, {sc.p, sc.n}, c.stream);
  }
  if (timed) {
    pre.b = ev();
    sw.a = ev();
  }
  Train y;
  double f1 = 0.0, f2 = 0.0;
  for (int k = 0; k < K; ++k) {
    const Core &a = A.cores[k], &v = x.cores[k];
    Core yk = make_core(c, v.r0, a.m, 1, v.r1);
    const EnvBuf& pr = R[k + 1];
    EvPair e1;
    if (timed && split_timing) e1.a = ev();
    local_matvec(L.d.p, L.b, L.o, L.k, A.Ap[k].p, a.m, a.n, a.r1, pr.d.p, pr.b, pr.k, v.d.p, yk.d.p, 1.0, 0.0,
                 {sc.p, sc.n}, c.stream);
    if (timed && split_timing) {
      e1.b = ev();
      k1.push_back(e1);
    }
    f1 += local_matvec_flops(L.b, L.o, L.k, a.m, a.n, a.r1, pr.b, pr.k);
    y.cores.push_back(std::move(yk));
    if (k + 1 < K) {
      EnvBuf nl;
      nl.b = v.r1; nl.o = a.r1; nl.k = v.r1;
      nl.d.alloc((long long)nl.b * nl.o * nl.k, c.stream);
      EvPair e2;
      if (timed && split_timing) e2.a = ev();
      env_left(L.d.p, L.b, L.o, L.k, v.d.p, v.r1, A.Ap[k].p, a.m, a.n, a.r1, v.d.p, v.r1, nl.d.p, {sc.p, sc.n},
               c.stream);
      if (timed && split_timing) {
        e2.b = ev();
        k2.push_back(e2);
      }
      f2 += env_flops(L.b, L.o, L.k, a.m, a.n, a.r1, v.r1, v.r1);
      L = std::move(nl);
    }
  }
  if (timed) {
    sw.b = ev();
    c.sync();
    *t = SweepTimes{};
    t->prepass_ms = elapsed(pre);
    t->sweep_ms = elapsed(sw);
    for (auto& e : k1) t->k1_ms += elapsed(e);
    for (auto& e : k2) t->k2_ms += elapsed(e);
    t->k1_flops = f1;
    t->k2_flops = f2;
    double fr = 0.0;
    for (int k = K - 1; k >= 1; --k) {
      const Core &a = A.cores[k], &v = x.cores[k];
      fr += env_flops(R[k + 1].b, R[k + 1].o, R[k + 1].k, a.m, a.n, a.r0, v.r0, v.r0);
    }
    t->prepass_flops = fr;
  }
  for (auto e : evs) QTT_CUDA(cudaEventDestroy(e));
  return y;
}

}  // namespace qtt
