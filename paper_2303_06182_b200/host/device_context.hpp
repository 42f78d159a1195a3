// Process-wide C-ABI context shared by the moesim:: drop-in functions
// (gating, exchange planning, cache policy).  Internal to libmoesim_b200.
//
// The C ABI context is not thread-safe, so every call made through
// with_context() holds one mutex; the reference API is free functions with
// no handle, hence the single lazily created context on device 0.  Without a
// usable B200 the first call throws std::runtime_error (no CPU fallback).
#pragma once

#include <mutex>
#include <string>

#include "moe_capi.h"

namespace moesim::detail {

std::mutex& context_mutex();
moe_ctx* context_locked();  // caller holds context_mutex()

/// MOE_ERR_INVALID_ARGUMENT -> std::invalid_argument(message), anything else
/// -> std::runtime_error.
[[noreturn]] void rethrow(int status);

/// Runs fn(ctx) -> moe_status under the lock; throws on a non-OK status.
template <class F>
void with_context(F&& fn) {
  std::lock_guard<std::mutex> lock(context_mutex());
  const int st = fn(context_locked());
  if (st != MOE_OK) rethrow(st);
}

}  // namespace moesim::detail
