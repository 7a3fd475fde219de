// FP64 tensor-core GEMM for sm_100a: warp-level DMMA (mma.sync m8n8k4 f64),
// cp.async multi-stage shared-memory pipeline, arbitrary operand strides and a
// two-level batch index.  This is the workhorse under every TT contraction of
// the AMEn sweep (local matvec, environment updates, dense local matrix) and the
// blocked dense kernels (Cholesky trailing update, QR block reflectors).
//
// Operand convention (all element strides, in doubles):
//   op(A)(i,k) = A[i*a_rs + k*a_cs + b1*a_bs1 + b2*a_bs2]        i < M, k < K
//   op(B)(k,j) = B[k*b_rs + j*b_cs + b1*b_bs1 + b2*b_bs2]        k < K, j < N
//   C(i,j)     = C[i*c_rs + j*c_cs + b1*c_bs1 + b2*c_bs2]
//   C = alpha * op(A) op(B) + beta * C       (beta == 0: C is not read)
// Transposes are just swapped strides, so one kernel covers NN/NT/TN/TT.
//
// sm_100a has no f64 tcgen05 kind (CUDA 12.9 tcgen05.mma kinds: f16, tf32,
// f8f6f4, i8, mxf8f6f4, mxf4, mxf4nvf4), so DMMA is the FP64 tensor path; SASS
// shows DMMA.8x8x4.  Measured peak on B200: 37.1 TF/s (profiles/fp64_peaks_r01.jsonl).
#pragma once
#include "common.cuh"

namespace qtt {

struct GemmArgs {
  int M = 0, N = 0, K = 0;
  const double* A = nullptr;
  long long a_rs = 0, a_cs = 0, a_bs1 = 0, a_bs2 = 0;
  const double* B = nullptr;
  long long b_rs = 0, b_cs = 0, b_bs1 = 0, b_bs2 = 0;
  double* C = nullptr;
  long long c_rs = 0, c_cs = 0, c_bs1 = 0, c_bs2 = 0;
  int batch1 = 1, batch2 = 1;
  double alpha = 1.0, beta = 0.0;
  // Optional device flag: when non-null and *skip != 0 the launch is a no-op
  // (device-resident CG loops stop without a host round trip).
  const int* skip = nullptr;
  // Only tiles touching the lower triangle (row >= col) are computed (SYRK-style
  // trailing update of the blocked Cholesky); strictly-upper tiles are skipped.
  bool lower_only = false;
};

// Row-major helpers: X is (rows x cols) with leading dimension ld.
inline void gemm_set_A(GemmArgs& g, const double* A, long long ld, bool trans) {
  g.A = A;
  if (!trans) { g.a_rs = ld; g.a_cs = 1; } else { g.a_rs = 1; g.a_cs = ld; }
}
inline void gemm_set_B(GemmArgs& g, const double* B, long long ld, bool trans) {
  g.B = B;
  if (!trans) { g.b_rs = ld; g.b_cs = 1; } else { g.b_rs = 1; g.b_cs = ld; }
}
inline void gemm_set_C(GemmArgs& g, double* C, long long ld) { g.C = C; g.c_rs = ld; g.c_cs = 1; }

// Launch (stream-ordered).  workspace may be null; when provided (>= ws_doubles)
// long-K products with few output tiles are split along K and reduced in a fixed
// order (deterministic).
void gemm(const GemmArgs& g, cudaStream_t s, double* workspace = nullptr, long long ws_doubles = 0);

// Scratch doubles gemm() would like for split-K of this shape (0 if not split).
long long gemm_workspace_hint(const GemmArgs& g);

}  // namespace qtt
