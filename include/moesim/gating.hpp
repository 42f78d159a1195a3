// Drop-in replacement for the reference's routing API
// (proj/include/moesim/gating.hpp), executed on a B200.
//
// Declarations, struct layouts and exception behaviour match the reference so
// code written against it -- including its own unit tests
// (proj/tests/test_gating.cpp, compiled unmodified against this header, see
// tests/test_route_gpu.py::test_reference_test_gating_compiled_against_dropin and
// tests/test_dropin_suites.py) -- builds and passes unchanged.  The work is
// done by the sm_100a kernels behind the C ABI (include/moe_capi.h):
//
//   dynamic_dispatch  -> moe_dynamic_dispatch_host  (stable counting sort)
//   static_dispatch   -> moe_static_dispatch_host   (rank + capacity clip)
//   combine<T>        -> moe_inverse_order_host     (inverse permutation)
//
// The CUDA device used is the current one when the first call is made (a
// process-wide context, guarded by a mutex).  Without a B200 every call throws
// std::runtime_error -- there is no CPU fallback.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <Eigen/Core>

#include "moesim/trace.hpp"

namespace moesim {

enum class GatingMode { kStatic, kDynamic };

struct GatingConfig {
  int num_experts = 0;
  int top_k = 1;
  double capacity_factor = 1.0;  // static mode only
  GatingMode mode = GatingMode::kDynamic;
};

inline constexpr int kPlaceholder = -1;

// ceil(C * S), snapping products within 1e-9 (relative) of an integer.
int expert_capacity(double capacity_factor, int seq_len);

// Capacity-factor routing: slots(e, c) holds the slot id t*k+j of the c-th
// assignment accepted by expert e (first come, first served in slot order)
// or kPlaceholder; overflowing assignments are listed in `dropped`.
struct StaticDispatchPlan {
  int seq_len = 0;
  int num_experts = 0;
  int top_k = 1;
  int capacity = 0;
  Eigen::MatrixXi slots;                     // num_experts x capacity
  std::vector<std::pair<int, int>> dropped;  // (token, expert)

  int placed() const { return static_cast<int>((slots.array() != kPlaceholder).count()); }
};

// Dynamic gating: every slot id grouped by expert, ascending inside a group.
// order[splits[e] .. splits[e+1]) are expert e's slots; nothing is dropped.
struct DynamicDispatchPlan {
  int seq_len = 0;
  int num_experts = 0;
  int top_k = 1;
  std::vector<int> order;
  std::vector<int> counts;
  std::vector<int> splits;
};

struct WasteFactor {
  double value = 0.0;
};

StaticDispatchPlan static_dispatch(const Batch& batch, const GatingConfig& cfg);
DynamicDispatchPlan dynamic_dispatch(const Batch& batch, const GatingConfig& cfg);

// E * C / k: provisioned slots over real assignments.
WasteFactor waste_factor(int num_experts, double capacity_factor, int top_k);

// Elements of the (E, S, capacity) one-hot dispatch mask static gating implies.
std::int64_t dispatch_mask_elements(int seq_len, int num_experts, double capacity_factor);

struct DispatchCostCounts {
  std::int64_t comparisons = 0;
  std::int64_t count_passes = 0;
  std::int64_t gather_elements = 0;
};

DispatchCostCounts dispatch_cost_counts(const DynamicDispatchPlan& plan, int token_dim);

std::string debug_json(const StaticDispatchPlan& plan);
std::string debug_json(const DynamicDispatchPlan& plan);

template <typename T>
struct CombinedEntry {
  int expert = 0;
  double weight = 0.0;
  T payload{};
};

template <typename T>
using CombinedBatch = std::vector<std::vector<CombinedEntry<T>>>;

namespace detail {
// GPU inverse permutation: pos[order[p]] = p (order entries of -1 skipped),
// pos sized n_slots and pre-filled with -1.
std::vector<int> inverse_order(const int* order, std::int64_t n, std::int64_t n_slots);
}  // namespace detail

// Dynamic combine: outputs[p] is the payload produced for plan.order[p]; each
// token gets its k entries back in assignment-slot order.
template <typename T>
CombinedBatch<T> combine(const DynamicDispatchPlan& plan, const Batch& batch,
                         std::span<const T> outputs) {
  const int k = plan.top_k;
  const std::int64_t n = static_cast<std::int64_t>(plan.seq_len) * k;
  if (static_cast<std::int64_t>(outputs.size()) != n)
    throw std::invalid_argument("combine: payload count mismatch vs. plan");
  if (batch.seq_len() != plan.seq_len)
    throw std::invalid_argument("combine: batch does not match plan");
  const std::vector<int> pos = detail::inverse_order(plan.order.data(), n, n);
  CombinedBatch<T> result(static_cast<std::size_t>(plan.seq_len));
  for (int t = 0; t < plan.seq_len; ++t) {
    const TokenAssignment& ta = batch.tokens[static_cast<std::size_t>(t)];
    auto& entries = result[static_cast<std::size_t>(t)];
    entries.reserve(static_cast<std::size_t>(k));
    for (int j = 0; j < k; ++j) {
      const int p = pos[static_cast<std::size_t>(t) * k + j];
      entries.push_back(CombinedEntry<T>{ta.experts[static_cast<std::size_t>(j)],
                                         ta.weights[static_cast<std::size_t>(j)],
                                         outputs[static_cast<std::size_t>(p)]});
    }
  }
  return result;
}

// Static combine: outputs is expert-major, one payload per capacity slot
// (E * capacity); placeholders are never delivered, dropped assignments
// deliver nothing, so a token may receive fewer than k entries.
template <typename T>
CombinedBatch<T> combine(const StaticDispatchPlan& plan, const Batch& batch,
                         std::span<const T> outputs) {
  const int k = plan.top_k;
  const std::int64_t cells = static_cast<std::int64_t>(plan.num_experts) * plan.capacity;
  if (static_cast<std::int64_t>(outputs.size()) != cells)
    throw std::invalid_argument("combine: payload count mismatch vs. plan");
  if (batch.seq_len() != plan.seq_len)
    throw std::invalid_argument("combine: batch does not match plan");
  std::vector<int> flat(static_cast<std::size_t>(cells));
  for (int e = 0; e < plan.num_experts; ++e)
    for (int c = 0; c < plan.capacity; ++c)
      flat[static_cast<std::size_t>(e) * plan.capacity + c] = plan.slots(e, c);
  const std::int64_t n = static_cast<std::int64_t>(plan.seq_len) * k;
  const std::vector<int> pos = detail::inverse_order(flat.data(), cells, n);
  CombinedBatch<T> result(static_cast<std::size_t>(plan.seq_len));
  for (int t = 0; t < plan.seq_len; ++t) {
    const TokenAssignment& ta = batch.tokens[static_cast<std::size_t>(t)];
    for (int j = 0; j < k; ++j) {
      const int p = pos[static_cast<std::size_t>(t) * k + j];
      if (p < 0) continue;
      result[static_cast<std::size_t>(t)].push_back(
          CombinedEntry<T>{p / plan.capacity, ta.weights[static_cast<std::size_t>(j)],
                           outputs[static_cast<std::size_t>(p)]});
    }
  }
  return result;
}

}  // namespace moesim
