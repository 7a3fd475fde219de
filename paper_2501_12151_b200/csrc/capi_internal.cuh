// Opaque C-ABI handle types shared by the capi*.cu translation units.
#pragma once
#include "engine.cuh"
#include "train.cuh"

struct qtt_ctx {
  qtt::Ctx impl;
  explicit qtt_ctx(int dev) : impl(dev) {}
};

struct qtt_train {
  qtt::Train t;
};

namespace qtt {
// Records the message for qtt_last_error() and returns code (capi.cu).
int capi_guard_store(const char* what, int code);
}  // namespace qtt
