// Synthetic skewed routing (include/moesim/trace.hpp: gen_synthetic_trace).
//
// Workload generator only -- it produces TokenAssignment lists that the GPU
// layer consumes through moe_layer_forward_routed / moe_cache_forward_routed.
// The random stream is consumed in the same order as the reference generator
// (proj/src/trace.cpp:174-259), so a given spec yields the same trace bit for
// bit (checked against the verbatim reference build in tests/test_trace_gen.py).
#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "moesim/trace.hpp"

namespace moesim {

namespace {

// 53 random mantissa bits -> [0, 1)
double draw_unit(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

// Uniform integer in [0, n): reject the biased tail of the 64-bit range.
std::uint64_t draw_below(std::mt19937_64& g, std::uint64_t n) {
  const std::uint64_t top = std::numeric_limits<std::uint64_t>::max();
  const std::uint64_t cutoff = top - top % n;
  for (;;) {
    const std::uint64_t v = g();
    if (v < cutoff) return v % n;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

}  // namespace

TokenTrace gen_synthetic_trace(const SyntheticSpec& spec) {
  require(spec.num_experts >= 1, "num_experts must be positive");
  require(spec.top_k >= 1, "top_k must be positive");
  require(spec.num_batches >= 1, "num_batches must be positive");
  require(spec.seq_len >= 1, "seq_len must be positive");
  require(spec.zipf_skew >= 0.0, "zipf_skew must be >= 0");
  require(spec.persistence >= 0.0 && spec.persistence <= 1.0, "persistence must be in [0, 1]");
  require(spec.active_fraction > 0.0 && spec.active_fraction <= 1.0,
          "active_fraction must be in (0, 1]");
  const int E = spec.num_experts;
  const int hot = static_cast<int>(std::ceil(spec.active_fraction * E));
  require(hot >= spec.top_k, "not enough active experts for top-k");

  std::mt19937_64 g(spec.seed);
  // popularity of the r-th ranked hot expert, and the total mass
  std::vector<double> mass(static_cast<std::size_t>(hot));
  double total = 0.0;
  for (int r = 0; r < hot; ++r) mass[static_cast<std::size_t>(r)] = std::pow(r + 1.0, -spec.zipf_skew);
  for (int r = 0; r < hot; ++r) total += mass[static_cast<std::size_t>(r)];

  // ranked[r] = expert holding popularity rank r (first `hot` entries)
  std::vector<int> ranked(static_cast<std::size_t>(E));
  for (int e = 0; e < E; ++e) ranked[static_cast<std::size_t>(e)] = e;
  auto shuffle_hot = [&]() {
    for (int r = 0; r < hot; ++r) {
      const int pick = r + static_cast<int>(draw_below(g, static_cast<std::uint64_t>(E - r)));
      std::swap(ranked[static_cast<std::size_t>(r)], ranked[static_cast<std::size_t>(pick)]);
    }
  };
  shuffle_hot();

  TokenTrace out;
  out.num_experts = E;
  out.top_k = spec.top_k;
  out.batches.resize(static_cast<std::size_t>(spec.num_batches));
  std::vector<char> used(static_cast<std::size_t>(hot));
  for (int b = 0; b < spec.num_batches; ++b) {
    if (b > 0 && draw_unit(g) >= spec.persistence) shuffle_hot();
    Batch& batch = out.batches[static_cast<std::size_t>(b)];
    batch.batch_id = b;
    batch.tokens.resize(static_cast<std::size_t>(spec.seq_len));
    for (TokenAssignment& ta : batch.tokens) {
      std::fill(used.begin(), used.end(), 0);
      double left = total;
      for (int j = 0; j < spec.top_k; ++j) {
        const double target = draw_unit(g) * left;
        int pick = -1;
        double run = 0.0;
        for (int r = 0; r < hot && pick < 0; ++r) {
          if (used[static_cast<std::size_t>(r)]) continue;
          run += mass[static_cast<std::size_t>(r)];
          if (target < run) pick = r;
        }
        for (int r = hot - 1; pick < 0 && r >= 0; --r)  // rounding: last unused rank
          if (!used[static_cast<std::size_t>(r)]) pick = r;
        used[static_cast<std::size_t>(pick)] = 1;
        left -= mass[static_cast<std::size_t>(pick)];
        ta.experts.push_back(ranked[static_cast<std::size_t>(pick)]);
      }
      double sum = 0.0;
      for (int j = 0; j < spec.top_k; ++j) {
        ta.weights.push_back(draw_unit(g) + 1e-12);
        sum += ta.weights.back();
      }
      for (double& x : ta.weights) x /= sum;
    }
  }
  return out;
}

}  // namespace moesim

// Flat form for the Python host (paper_2303_06182_b200/traces.py):
// experts/weights are [num_batches, seq_len, top_k].  Returns 0, or 1 with the
// reference's std::invalid_argument text in `err`.
extern "C" int moesim_gen_synthetic_routing(int E, int k, int B, int S, double skew,
                                            double persistence, double active_fraction,
                                            std::uint64_t seed, int* experts, double* weights,
                                            char* err, int err_len) {
  try {
    moesim::SyntheticSpec spec{E, k, B, S, skew, persistence, active_fraction, seed};
    const moesim::TokenTrace tr = moesim::gen_synthetic_trace(spec);
    std::size_t i = 0;
    for (const auto& batch : tr.batches)
      for (const auto& ta : batch.tokens)
        for (int j = 0; j < k; ++j, ++i) {
          experts[i] = ta.experts[static_cast<std::size_t>(j)];
          weights[i] = ta.weights[static_cast<std::size_t>(j)];
        }
    return 0;
  } catch (const std::exception& e) {
    if (err && err_len > 0) {
      std::string m = e.what();
      m.resize(std::min<std::size_t>(m.size(), static_cast<std::size_t>(err_len - 1)));
      std::copy(m.begin(), m.end(), err);
      err[m.size()] = 0;
    }
    return 1;
  }
}
