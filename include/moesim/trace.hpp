// Routing-decision types of the MoE layer, source-compatible with the
// reference's proj/include/moesim/trace.hpp:15-45 (same names, field names and
// field order -- tests aggregate-initialise them, e.g. TokenAssignment{{e},{1.0}}).
//
// Only the types the dispatch path consumes are provided.  The reference's
// trace I/O, synthetic generator and statistics (trace.hpp:52-96) are
// simulator tooling outside this library's scope.
#pragma once

#include <cstdint>
#include <vector>

#include <Eigen/Core>

namespace moesim {

// Top-k routing decision of one token: k distinct expert ids in [0, E) and
// gate weights >= 0 summing to 1 (reference invariants, trace.cpp:47-67).
// On the GPU path these come from the gate kernel (moe_gate_topk).
struct TokenAssignment {
  std::vector<int> experts;
  std::vector<double> weights;
};

// One layer call's flattened tokens (S = batch x sequence).
struct Batch {
  std::int64_t batch_id = 0;
  std::vector<TokenAssignment> tokens;

  int seq_len() const { return static_cast<int>(tokens.size()); }
};

struct TokenTrace {
  int num_experts = 0;
  int top_k = 0;
  std::vector<Batch> batches;

  int num_batches() const { return static_cast<int>(batches.size()); }
};

// Synthetic routing workload (reference trace.hpp:52-61): per batch, Zipf(skew)
// popularity over a random subset of ceil(active_fraction * E) experts, kept
// for the next batch with probability `persistence`; each token draws k
// distinct experts proportionally to popularity.  Used here to drive skewed
// routing into the GPU layer (expert-cache workloads, trace replay).
struct SyntheticSpec {
  int num_experts = 0;
  int top_k = 1;
  int num_batches = 1;
  int seq_len = 1;
  double zipf_skew = 0.0;
  double persistence = 0.0;
  double active_fraction = 1.0;
  std::uint64_t seed = 0;
};

// Deterministic for a given spec; bit-identical to the reference generator
// (same std::mt19937_64 stream, trace.cpp:174-259; tests/test_trace_gen.py).
TokenTrace gen_synthetic_trace(const SyntheticSpec& spec);

// Expert x batch load shares (each column sums to 1).
struct LoadMatrix {
  Eigen::MatrixXd share;

  Eigen::Index num_experts() const { return share.rows(); }
  Eigen::Index num_batches() const { return share.cols(); }
};

}  // namespace moesim
