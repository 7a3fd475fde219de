// Config-4 microbench operation: right-env pre-pass + one L->R sweep of
// local matvecs and left environment updates (amen.py:108-137), all device-resident.
#pragma once
#include "train.cuh"

namespace qtt {

struct SweepTimes {
  double prepass_ms = 0, sweep_ms = 0;  // wall (CUDA events) of the pre-pass / the sweep
  double k1_ms = 0, k2_ms = 0;          // summed per-launch-group times (split_timing only)
  double k1_flops = 0, k2_flops = 0;    // algorithmic flops of the sweep's K1 / K2 calls
  double prepass_flops = 0;             // right-environment pre-pass flops
};

// Returns y with y_k = local matvec at core k (shape (r_{k-1}, m_k, r_k)).  t may be null.
Train matvec_sweep(Ctx& c, Train& A, const Train& x, SweepTimes* t, bool split_timing);

}  // namespace qtt
