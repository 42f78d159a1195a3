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

// Expert x batch load shares (each column sums to 1).
struct LoadMatrix {
  Eigen::MatrixXd share;

  Eigen::Index num_experts() const { return share.rows(); }
  Eigen::Index num_batches() const { return share.cols(); }
};

}  // namespace moesim
