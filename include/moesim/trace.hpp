// Routing-decision types of the MoE layer, source-compatible with the
// reference's proj/include/moesim/trace.hpp:15-45 (same names, field names and
// field order -- tests aggregate-initialise them, e.g. TokenAssignment{{e},{1.0}}).
//
// Besides the types: the synthetic generator, the JSON Lines trace files and
// the invariant checker / load matrix of the reference (trace.hpp:52-88), so
// generated or recorded routing can be replayed through the GPU layer
// (tools/moesim_measure --trace), and the load-matrix utilities the
// placement protocol uses (split_trace, sparsity_stats, CSV export).
#pragma once

#include <cstdint>
#include <filesystem>
#include <utility>
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

/// Checks every trace invariant (k distinct ids in [0, E), weights >= 0
/// summing to 1, strictly increasing batch ids, non-empty batches); throws
/// std::invalid_argument naming the batch/token of the first violation, with
/// the reference's message text (trace.cpp:47-87).
void validate(const TokenTrace& trace);

/// JSON Lines: header {"num_experts","top_k","version":1}, then one line per
/// batch.  load throws std::runtime_error (I/O, parse) or std::invalid_argument
/// (invariants) with file:line context; save is byte-deterministic and writes
/// the same bytes as the reference for the same trace.
TokenTrace load_token_trace(const std::filesystem::path& path);
void save_token_trace(const TokenTrace& trace, const std::filesystem::path& path);

/// share(e, b) = fraction of batch b's k * seq_len slots routed to expert e.
LoadMatrix aggregate_loads(const TokenTrace& trace);

struct SparsityReport {
  std::vector<int> inactive_per_batch;      // experts with zero share, per batch
  std::vector<double> top_share_per_batch;  // largest single-expert share
  Eigen::VectorXd mean_load;                // per-expert mean over batches
  double mean_inactive_fraction = 0.0;
  double max_inactive_fraction = 0.0;
  int never_active = 0;  // experts with zero share in every batch
};

/// Batch columns [0, cut) and [cut, B), cut = floor(fraction * B) (snapped
/// when within 1e-9 of an integer); std::invalid_argument if a part is empty.
std::pair<LoadMatrix, LoadMatrix> split_trace(const LoadMatrix& loads, double fraction);

SparsityReport sparsity_stats(const LoadMatrix& loads);

/// CSV "expert,b0,b1,..." with one row per expert (doubles as %.12g).
void save_load_matrix_csv(const LoadMatrix& loads, const std::filesystem::path& path);

}  // namespace moesim
