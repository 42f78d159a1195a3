// Routing-trace files and load statistics (include/moesim/trace.hpp): the
// reference's JSON Lines trace format (proj/include/moesim/trace.hpp:63-70,
// proj/src/trace.cpp:89-157) so recorded or generated traces can be replayed
// through the GPU layer (tools/moesim_measure --trace), plus the invariant
// checker and the expert x batch load matrix (trace.cpp:47-87,158-172).
//
// Format: a header {"num_experts":E,"top_k":k,"version":1}, then one line per
// batch {"batch_id":b,"tokens":[{"e":[...],"w":[...]},...]}; keys sorted
// (nlohmann json's default object), so a trace saves to the same bytes as the
// reference writes (tests/test_trace_io.py).
#include <cmath>
#include <cstdint>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "moesim/trace.hpp"

namespace moesim {

namespace {

using nlohmann::json;

[[noreturn]] void invalid(const std::string& what) { throw std::invalid_argument(what); }

std::string where(int batch_id, int token) {
  return " (batch " + std::to_string(batch_id) + ", token " + std::to_string(token) + ")";
}

// k distinct ids in [0, E), weights >= 0 summing to 1 within 1e-9.
void check_token(const TokenAssignment& ta, int E, int k, int b, int t) {
  const std::size_t n = ta.experts.size();
  if (static_cast<int>(n) != k)
    invalid("expected " + std::to_string(k) + " experts per token" + where(b, t));
  if (ta.weights.size() != n) invalid("weights/experts length mismatch" + where(b, t));
  double total = 0.0;
  for (std::size_t j = 0; j < n; ++j) {
    const int e = ta.experts[j];
    if (e < 0 || e >= E)
      invalid("expert id " + std::to_string(e) + " out of range [0, " + std::to_string(E) + ")" +
              where(b, t));
    for (std::size_t i = j + 1; i < n; ++i)
      if (ta.experts[i] == e) invalid("duplicate expert in top-k" + where(b, t));
    if (ta.weights[j] < 0.0) invalid("negative gate weight" + where(b, t));
    total += ta.weights[j];
  }
  if (std::abs(total - 1.0) > 1e-9) invalid("weights do not sum to 1" + where(b, t));
}

}  // namespace

void validate(const TokenTrace& trace) {
  if (trace.num_experts < 1) invalid("num_experts must be positive");
  if (trace.top_k < 1) invalid("top_k must be positive");
  if (trace.top_k > trace.num_experts) invalid("top_k exceeds num_experts");
  std::int64_t last = -1;
  for (const Batch& b : trace.batches) {
    if (b.batch_id < 0) invalid("negative batch_id " + std::to_string(b.batch_id));
    if (b.batch_id <= last)
      invalid("batch_ids not strictly increasing at batch " + std::to_string(b.batch_id));
    last = b.batch_id;
    if (b.tokens.empty()) invalid("batch " + std::to_string(b.batch_id) + " has no tokens");
    for (int t = 0; t < b.seq_len(); ++t)
      check_token(b.tokens[static_cast<std::size_t>(t)], trace.num_experts, trace.top_k,
                  static_cast<int>(b.batch_id), t);
  }
}

TokenTrace load_token_trace(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open trace file: " + path.string());
  const std::string name = path.string();
  TokenTrace trace;
  bool header = false;
  std::string line;
  for (int no = 1; std::getline(in, line); ++no) {
    if (line.empty()) continue;
    const std::string at = name + ":" + std::to_string(no) + ": ";
    json rec;
    try {
      rec = json::parse(line);
    } catch (const json::parse_error& e) {
      throw std::runtime_error(at + "parse error: " + e.what());
    }
    try {
      if (!header) {
        if (rec.value("version", 0) != 1) throw std::runtime_error(at + "unsupported trace version");
        trace.num_experts = rec.at("num_experts").get<int>();
        trace.top_k = rec.at("top_k").get<int>();
        header = true;
        continue;
      }
      Batch b;
      b.batch_id = rec.at("batch_id").get<std::int64_t>();
      const json& toks = rec.at("tokens");
      b.tokens.reserve(toks.size());
      for (const json& tj : toks)
        b.tokens.push_back(
            TokenAssignment{tj.at("e").get<std::vector<int>>(), tj.at("w").get<std::vector<double>>()});
      trace.batches.push_back(std::move(b));
    } catch (const json::exception& e) {
      throw std::runtime_error(at + "malformed record: " + e.what());
    }
  }
  if (!header) throw std::runtime_error(name + ": empty trace (missing header line)");
  try {
    validate(trace);
  } catch (const std::invalid_argument& e) {
    throw std::invalid_argument(name + ": " + e.what());
  }
  return trace;
}

void save_token_trace(const TokenTrace& trace, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write trace file: " + path.string());
  out << json{{"version", 1}, {"num_experts", trace.num_experts}, {"top_k", trace.top_k}}.dump()
      << '\n';
  for (const Batch& b : trace.batches) {
    json toks = json::array();
    for (const TokenAssignment& ta : b.tokens) toks.push_back({{"e", ta.experts}, {"w", ta.weights}});
    out << json{{"batch_id", b.batch_id}, {"tokens", std::move(toks)}}.dump() << '\n';
  }
}

LoadMatrix aggregate_loads(const TokenTrace& trace) {
  validate(trace);
  LoadMatrix L;
  const int E = trace.num_experts, B = trace.num_batches();
  L.share = Eigen::MatrixXd::Zero(E, B);
  for (int b = 0; b < B; ++b) {
    // integer slot counts, then one division per entry (exact counts / k*S)
    const Batch& batch = trace.batches[static_cast<std::size_t>(b)];
    for (const TokenAssignment& ta : batch.tokens)
      for (int e : ta.experts) L.share(e, b) += 1.0;
    const double slots = static_cast<double>(trace.top_k) * batch.seq_len();
    for (int e = 0; e < E; ++e) L.share(e, b) /= slots;
  }
  return L;
}

}  // namespace moesim

// ---- flat C entry points for the host tests (tests/test_trace_io.py) ------
namespace {
int report(const std::exception& e, char* err, int err_len) {
  if (err && err_len > 0) {
    std::string m = e.what();
    if (m.size() >= static_cast<std::size_t>(err_len)) m.resize(static_cast<std::size_t>(err_len - 1));
    std::copy(m.begin(), m.end(), err);
    err[m.size()] = 0;
  }
  return dynamic_cast<const std::invalid_argument*>(&e) ? 1 : 2;
}
}  // namespace

// Generate a synthetic trace and save it (JSON Lines).  0 / 1 invalid_argument / 2 other.
extern "C" int moesim_save_synthetic_trace(int E, int k, int B, int S, double skew,
                                           double persistence, double active_fraction,
                                           std::uint64_t seed, const char* path, char* err,
                                           int err_len) {
  try {
    moesim::SyntheticSpec spec{E, k, B, S, skew, persistence, active_fraction, seed};
    moesim::save_token_trace(moesim::gen_synthetic_trace(spec), path);
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, err_len);
  }
}

// Load (validating) and save again; dims[0..2] = E, k, batches.
extern "C" int moesim_trace_roundtrip(const char* in_path, const char* out_path, int* dims,
                                      char* err, int err_len) {
  try {
    const moesim::TokenTrace tr = moesim::load_token_trace(in_path);
    if (dims) {
      dims[0] = tr.num_experts;
      dims[1] = tr.top_k;
      dims[2] = tr.num_batches();
    }
    if (out_path && *out_path) moesim::save_token_trace(tr, out_path);
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, err_len);
  }
}

// Load shares [E, B] (column-major, as Eigen) of a trace file.
extern "C" int moesim_trace_loads(const char* path, double* share, int cap, char* err, int err_len) {
  try {
    const moesim::LoadMatrix L = moesim::aggregate_loads(moesim::load_token_trace(path));
    const long n = static_cast<long>(L.share.rows()) * L.share.cols();
    if (n > cap) throw std::runtime_error("load buffer too small");
    for (long i = 0; i < n; ++i) share[i] = L.share.data()[i];
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, err_len);
  }
}
