// Shared helpers for the QTT engine (sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace qtt {

// Error categories mirror ttfem/errors.py:9-34 (mapped in the C-ABI to status codes).
enum Status : int {
  QTT_OK = 0,
  QTT_ERR_SHAPE = 1,     // ShapeMismatchError
  QTT_ERR_SOLVER = 2,    // SolverError
  QTT_ERR_CAPACITY = 3,  // CapacityError (device OOM)
  QTT_ERR_CUDA = 4,      // CUDA runtime failure
  QTT_ERR_ARG = 5,       // invalid argument (ValueError)
};

struct Error : public std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define QTT_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      int _c = (_e == cudaErrorMemoryAllocation) ? ::qtt::QTT_ERR_CAPACITY : ::qtt::QTT_ERR_CUDA; \
      throw ::qtt::Error(_c, std::string(#expr " failed: ") + cudaGetErrorString(_e) +     \
                                 " at " __FILE__ ":" + std::to_string(__LINE__));          \
    }                                                                                      \
  } while (0)

#define QTT_CHECK_LAUNCH()           \
  do {                               \
    QTT_CUDA(cudaGetLastError());    \
    ::qtt::count_launch();           \
  } while (0)

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// Per-device one-time state (kernel function attributes and occupancy-derived grid sizes are
// per device; every C-ABI entry makes its context's device current first, capi.cu).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}
template <class T>
struct PerDevice {
  T v[kMaxDevices];
  explicit PerDevice(T init) {
    for (auto& x : v) x = init;
  }
  T& operator()() { return v[current_device()]; }
  T& at(int d) { return v[d >= 0 && d < kMaxDevices ? d : 0]; }
};

// Process-wide count of kernel launches issued by this library (reported as
// "gpu_launches" by bench.py; every launcher calls count_launch()).
long long launch_count();
void count_launch(long long n = 1);

}  // namespace qtt
