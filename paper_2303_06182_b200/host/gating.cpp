// moesim:: routing API (include/moesim/gating.hpp) on top of the C ABI.
//
// Host side only: argument checks with the reference's exact messages
// (proj/src/gating.cpp:13-17,33-42,61,90,96,102), flattening of Batch into
// the int32 slot layout the kernels consume, and re-assembly of the plans.
// The dispatch itself runs on the GPU (moe_*_dispatch_host).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "moe_capi.h"
#include "device_context.hpp"
#include "moesim/gating.hpp"

namespace moesim {

namespace {

using detail::with_context;

void check_batch(const Batch& batch, const GatingConfig& cfg) {
  if (cfg.num_experts < 1) throw std::invalid_argument("num_experts must be positive");
  if (cfg.top_k < 1) throw std::invalid_argument("top_k must be positive");
  if (cfg.top_k > cfg.num_experts) throw std::invalid_argument("top_k exceeds num_experts");
  if (batch.tokens.empty()) throw std::invalid_argument("empty batch");
}

std::vector<std::int32_t> flatten(const Batch& batch, int k) {
  std::vector<std::int32_t> ids(static_cast<std::size_t>(batch.seq_len()) * k);
  std::size_t i = 0;
  for (const TokenAssignment& ta : batch.tokens)
    for (int j = 0; j < k; ++j) ids[i++] = ta.experts[static_cast<std::size_t>(j)];
  return ids;
}

}  // namespace

namespace detail {

std::vector<int> inverse_order(const int* order, std::int64_t n, std::int64_t n_slots) {
  std::vector<int> pos(static_cast<std::size_t>(std::max<std::int64_t>(n_slots, 1)), -1);
  with_context([&](moe_ctx* c) { return moe_inverse_order_host(c, order, n, pos.data(), n_slots); });
  pos.resize(static_cast<std::size_t>(n_slots));
  return pos;
}

}  // namespace detail

int expert_capacity(double capacity_factor, int seq_len) {
  return moe_expert_capacity(capacity_factor, seq_len);
}

DynamicDispatchPlan dynamic_dispatch(const Batch& batch, const GatingConfig& cfg) {
  check_batch(batch, cfg);
  if (cfg.mode != GatingMode::kDynamic)
    throw std::invalid_argument("dynamic_dispatch requires dynamic mode");
  DynamicDispatchPlan plan;
  plan.seq_len = batch.seq_len();
  plan.num_experts = cfg.num_experts;
  plan.top_k = cfg.top_k;
  const std::vector<std::int32_t> ids = flatten(batch, cfg.top_k);
  plan.order.resize(ids.size());
  plan.counts.resize(static_cast<std::size_t>(cfg.num_experts));
  plan.splits.resize(static_cast<std::size_t>(cfg.num_experts) + 1);
  with_context([&](moe_ctx* c) {
    return moe_dynamic_dispatch_host(c, ids.data(), plan.seq_len, plan.top_k, plan.num_experts,
                                     plan.order.data(), plan.counts.data(), plan.splits.data());
  });
  return plan;
}

StaticDispatchPlan static_dispatch(const Batch& batch, const GatingConfig& cfg) {
  check_batch(batch, cfg);
  if (cfg.mode != GatingMode::kStatic)
    throw std::invalid_argument("static_dispatch requires static mode");
  if (cfg.capacity_factor <= 0.0)
    throw std::invalid_argument("capacity factor must be positive in static mode");
  StaticDispatchPlan plan;
  plan.seq_len = batch.seq_len();
  plan.num_experts = cfg.num_experts;
  plan.top_k = cfg.top_k;
  plan.capacity = expert_capacity(cfg.capacity_factor, plan.seq_len);
  if (plan.capacity <= 0) throw std::invalid_argument("zero capacity");
  const std::vector<std::int32_t> ids = flatten(batch, cfg.top_k);
  const std::int64_t cells = static_cast<std::int64_t>(plan.num_experts) * plan.capacity;
  std::vector<std::int32_t> slots(static_cast<std::size_t>(cells));
  std::vector<std::int32_t> dropped(2 * ids.size() + 2);
  std::int32_t cap = 0, n_dropped = 0;
  with_context([&](moe_ctx* c) {
    return moe_static_dispatch_host(c, ids.data(), plan.seq_len, plan.top_k, plan.num_experts,
                                    cfg.capacity_factor, &cap, slots.data(), cells, dropped.data(),
                                    &n_dropped);
  });
  // the C ABI returns the table expert-major; Eigen's storage is column-major
  plan.slots = Eigen::MatrixXi::Constant(plan.num_experts, plan.capacity, kPlaceholder);
  for (int e = 0; e < plan.num_experts; ++e)
    for (int c = 0; c < plan.capacity; ++c)
      plan.slots(e, c) = slots[static_cast<std::size_t>(e) * plan.capacity + c];
  plan.dropped.reserve(static_cast<std::size_t>(n_dropped));
  for (int i = 0; i < n_dropped; ++i) plan.dropped.emplace_back(dropped[2 * i], dropped[2 * i + 1]);
  return plan;
}

WasteFactor waste_factor(int num_experts, double capacity_factor, int top_k) {
  if (num_experts <= 0 || capacity_factor <= 0.0 || top_k <= 0)
    throw std::invalid_argument("waste_factor requires positive inputs");
  return WasteFactor{num_experts * capacity_factor / top_k};
}

std::int64_t dispatch_mask_elements(int seq_len, int num_experts, double capacity_factor) {
  if (seq_len <= 0 || num_experts <= 0 || capacity_factor <= 0.0)
    throw std::invalid_argument("dispatch_mask_elements requires positive inputs");
  return static_cast<std::int64_t>(num_experts) * seq_len *
         expert_capacity(capacity_factor, seq_len);
}

namespace {
// Comparator calls of std::stable_sort over `key` -- the reference's
// instrumentation (gating.cpp:108-118) measures exactly this.
std::int64_t stable_sort_comparisons(const std::vector<int>& key) {
  std::vector<int> idx(key.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::int64_t n = 0;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    ++n;
    return key[static_cast<std::size_t>(a)] < key[static_cast<std::size_t>(b)];
  });
  return n;
}
}  // namespace

DispatchCostCounts dispatch_cost_counts(const DynamicDispatchPlan& plan, int token_dim) {
  if (token_dim <= 0) throw std::invalid_argument("token_dim must be positive");
  const std::int64_t total = static_cast<std::int64_t>(plan.seq_len) * plan.top_k;
  std::vector<int> key(static_cast<std::size_t>(total), 0);
  for (int e = 0; e < plan.num_experts; ++e)
    for (int p = plan.splits[static_cast<std::size_t>(e)];
         p < plan.splits[static_cast<std::size_t>(e) + 1]; ++p)
      key[static_cast<std::size_t>(plan.order[static_cast<std::size_t>(p)])] = e;
  DispatchCostCounts c;
  c.comparisons = stable_sort_comparisons(key);
  c.count_passes = total;
  c.gather_elements = total * token_dim;
  return c;
}

namespace {
void put_array(std::ostringstream& os, const std::vector<int>& v) {
  os << '[';
  for (std::size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << v[i];
  os << ']';
}
}  // namespace

// Keys in lexicographic order, no whitespace -- the byte format the reference
// gets from nlohmann::json::dump() (gating.cpp:127-153).
std::string debug_json(const StaticDispatchPlan& plan) {
  std::ostringstream os;
  os << "{\"capacity\":" << plan.capacity << ",\"dropped\":[";
  for (std::size_t i = 0; i < plan.dropped.size(); ++i)
    os << (i ? "," : "") << '[' << plan.dropped[i].first << ',' << plan.dropped[i].second << ']';
  os << "],\"num_experts\":" << plan.num_experts << ",\"seq_len\":" << plan.seq_len
     << ",\"slots\":[";
  for (int e = 0; e < plan.num_experts; ++e) {
    os << (e ? "," : "") << '[';
    for (int c = 0; c < plan.capacity; ++c) os << (c ? "," : "") << plan.slots(e, c);
    os << ']';
  }
  os << "],\"top_k\":" << plan.top_k << '}';
  return os.str();
}

std::string debug_json(const DynamicDispatchPlan& plan) {
  std::ostringstream os;
  os << "{\"counts\":";
  put_array(os, plan.counts);
  os << ",\"num_experts\":" << plan.num_experts << ",\"order\":";
  put_array(os, plan.order);
  os << ",\"seq_len\":" << plan.seq_len << ",\"splits\":";
  put_array(os, plan.splits);
  os << ",\"top_k\":" << plan.top_k << '}';
  return os.str();
}

}  // namespace moesim

// Flat helper for the Python mirror (paper_2303_06182_b200/gating.py).
extern "C" std::int64_t moesim_stable_sort_comparisons(const int* key, int n) {
  return moesim::stable_sort_comparisons(std::vector<int>(key, key + std::max(n, 0)));
}
