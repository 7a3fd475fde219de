// Device-resident tensor trains and the TT algebra of the hot path (tt.py).
#pragma once
#include <vector>

#include "common.cuh"
#include "engine.cuh"

namespace qtt {

// One core.  Vector cores are (r0, m, 1, r1) -- same record shape as the reference's
// QTT1 container (serialize.py:10-14); operator cores are (r0, m, n, r1).
struct Core {
  int r0 = 1, m = 1, n = 1, r1 = 1;
  DBuf d;
  long long numel() const { return (long long)r0 * m * n * r1; }
};

struct Train {
  bool is_op = false;
  std::vector<Core> cores;
  // operator only: permuted copies for the contraction chains (contract.cuh)
  std::vector<DBuf> Ap, Aq;
  int order() const { return (int)cores.size(); }
  std::vector<int> ranks() const {  // (1, r_1, ..., r_K)
    std::vector<int> r{cores.empty() ? 1 : cores[0].r0};
    for (auto& c : cores) r.push_back(c.r1);
    return r;
  }
  std::vector<int> dims() const {  // vector modes / operator column modes
    std::vector<int> d;
    for (auto& c : cores) d.push_back(is_op ? c.n : c.m);
    return d;
  }
  std::vector<int> row_dims() const {
    std::vector<int> d;
    for (auto& c : cores) d.push_back(c.m);
    return d;
  }
  long long numel() const {
    long long s = 0;
    for (auto& c : cores) s += c.numel();
    return s;
  }
};

Core make_core(Ctx& c, int r0, int m, int n, int r1);
Train clone(Ctx& c, const Train& t);
void prepare_operator(Ctx& c, Train& A);  // builds Ap/Aq (idempotent)

// tt.py:396-406, in place: R->L thin QR; cores[1:] right-orthonormal afterwards.
void orthogonalize_rl(Ctx& c, Train& t);
// tt.py:362-371
double tt_norm(Ctx& c, const Train& t);
// tt.py:351-359
double tt_dot(Ctx& c, const Train& a, const Train& b);
// tt.py:409-429 (max_rank <= 0: uncapped)
Train tt_round(Ctx& c, const Train& a, double rel_tol, int max_rank);
// tt.py:434-449 with policy=None (Kronecker cores, no rounding)
Train tt_apply(Ctx& c, const Train& A, const Train& x);
// the same into preallocated output cores of the right shapes (one launch for <= 64 cores)
void tt_apply_into(Ctx& c, const Train& A, const Train& x, Train& y);
// tt.py:308-336
Train tt_sub(Ctx& c, const Train& a, const Train& b);
Train tt_scale_copy(Ctx& c, const Train& a, double s);
Train tt_ones(Ctx& c, const std::vector<int>& dims, double first_value = 1.0);
Train tt_zero(Ctx& c, const std::vector<int>& dims);

// ||A x - f|| / ||f|| (amen.py:87-99).  See amen.cu for how the optional rounding
// of the reference is honoured (it changes the norm by <= rel_tol relative).
double residual_norm(Ctx& c, const Train& A, const Train& x, const Train& f, bool* used_gram = nullptr);
// Exact path: tt_norm(tt_sub(tt_apply(A, x), f)) via the QR sweep.
double residual_norm_exact(Ctx& c, const Train& A, const Train& x, const Train& f);
// Diagnostic Gram estimate (fast, loses digits when ||A|| ||x|| >> ||Ax - f||).
double residual_norm_gram(Ctx& c, const Train& A, const Train& x, const Train& f);

// Dense bridges (tt.py:276-298): entries at count multi-indices (device int array, count x K,
// row-major) into out_dev; the full C-order vector (prod dims doubles) into out_dev.
void tt_entries(Ctx& c, const Train& t, const int* idx_dev, long long count, double* out_dev);
void tt_full(Ctx& c, const Train& t, double* out_dev);

// Rank rule of tt.py:386-393, bit-for-bit given the same singular values.
int rank_for_tolerance(const double* s, int n, double delta);

}  // namespace qtt
