// TMA-fed DMMA GEMM for K-contiguous operands (see gemm_tma.cu); gemm() routes eligible
// products here.
#pragma once
#include "gemm.cuh"

namespace qtt {

struct TmaGemmPlan {
  int tiles = 0, splits = 1, kt_per = 0;
};

bool gemm_tma_eligible(const GemmArgs& g);
TmaGemmPlan gemm_tma_plan(const GemmArgs& g);
long long gemm_tma_workspace(const GemmArgs& g);
// Runs the product and returns true, or returns false (nothing launched) when the shape,
// strides or workspace do not qualify.
bool gemm_tma(const GemmArgs& g, cudaStream_t s, double* ws, long long ws_doubles);

}  // namespace qtt
